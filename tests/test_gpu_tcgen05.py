"""tcgen05 descriptor conventions the fused edge kernels rely on, pinned on
the hardware through fcg_selftest_mma (kind::f16, fp32 accumulate in TMEM,
SWIZZLE_NONE core-matrix layouts):
  * LBO = core-matrix stride along K, SBO = stride along M/N, for K-major
    and MN-major operands alike;
  * an M=64 accumulator row m lives in TMEM lane 32*(m//16) + m%16.
Small-integer operands make the products exact, so equality is exact."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(M, N, K, a_mn, b_mn, seed=0, a_order=0):
    import torch
    from paper_2602_13140_b200 import _lib
    rng = np.random.default_rng(seed)
    A = rng.integers(-4, 5, size=(M, K)).astype(np.float16)
    B = rng.integers(-4, 5, size=(N, K)).astype(np.float16)
    dA = torch.as_tensor(A.view(np.int16)).cuda()
    dB = torch.as_tensor(B.view(np.int16)).cuda()
    dump = torch.zeros(128, N, dtype=torch.float32, device="cuda")
    lib = _lib.load()
    # swap=1 on an MN-major operand selects LBO=K stride / SBO=MN stride
    _lib.check(lib.fcg_selftest_mma(_lib.vp(dA), _lib.vp(dB), _lib.vp(dump), M, N, K, a_mn,
                                    a_order, a_mn, b_mn, 0, b_mn,
                                    C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    return A.astype(np.float64) @ B.astype(np.float64).T, dump.cpu().numpy()


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("K", [64, 128])
def test_m128(a_mn, b_mn, K):
    ref, dump = _run(128, 128, K, a_mn, b_mn)
    np.testing.assert_array_equal(dump, ref)


@pytest.mark.parametrize("a_mn,b_mn", [(0, 1), (1, 1)])
def test_m64_lane_map(a_mn, b_mn):
    ref, dump = _run(64, 128, 128, a_mn, b_mn)
    lanes = [32 * (m // 16) + m % 16 for m in range(64)]
    np.testing.assert_array_equal(dump[lanes], ref)


@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("N", [32, 128])
def test_a_operand_in_tmem(b_mn, N):
    # kind::f16 with A from TMEM (K-major): row m in lane m, element k in
    # column k/2, low half for even k
    ref, dump = _run(128, N, 128, 0, b_mn, a_order=2)
    np.testing.assert_array_equal(dump, ref)
