"""GPU counterparts of the reference's benchmark harness (bench.py): the
degree-skew aggregation report (bench.py:91-118, asserted by
test_acceptance.py:292-301), pipeline timing (bench.py:57-76) and the
replica x backend sweep with its CSV schema (bench.py:22-28, :121-192).
Times are CUDA-event device times (wall clock for run_bench cells, as the
reference measures them).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .engine import _torch
from .inputs import skewed_segments

BENCH_SCHEMA = ("system,N,E,replicas,fused,segred,quant,steps,ms_per_step,"
                "timestep_mol_per_s,ns_per_day,io_base_bytes,io_flash_bytes,"
                "io_ratio,peak_edge_alloc_bytes,speedup_vs_reference")
WALL_DERIVED_COLUMNS = ("ms_per_step", "timestep_mol_per_s", "ns_per_day",
                        "speedup_vs_reference")


def _device_ms(fn, repeats: int) -> float:
    torch = _torch()
    fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(repeats):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b))
    return float(np.median(times))


def degree_skew_report(n_segments: int = 2000, e: int = 200_000, d: int = 64,
                       repeats: int = 5, seed: int = 0) -> dict:
    """Aggregation time on fixed-E uniform vs power-law segment layouts:
    libfcg's chunked CSR segment reduce (asserted robust) and an atomic
    scatter-add (index_add_, reported only)."""
    torch = _torch()
    lib = _lib.load()
    rng = np.random.default_rng(seed)
    values = torch.as_tensor(rng.standard_normal((e, d)).astype(np.float32)).cuda()
    stream = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    out = {}
    for kind in ("uniform", "powerlaw"):
        ptr, dst = skewed_segments(n_segments, e, kind)
        dptr = torch.as_tensor(ptr).cuda()
        ddst = torch.as_tensor(dst).cuda()
        res = torch.empty(n_segments, d, device="cuda")
        wb = lib.fcg_segment_reduce_workspace_bytes(e, d, n_segments)
        ws = torch.empty(int(wb), dtype=torch.uint8, device="cuda")

        def seg():
            _lib.check(lib.fcg_segment_reduce(_lib.vp(values), e, d, _lib.vp(dptr), n_segments,
                                              _lib.vp(res), _lib.vp(ws), wb, stream()),
                       "fcg_segment_reduce")

        def scat():
            torch.zeros(n_segments, d, device="cuda").index_add_(0, ddst, values)

        out[kind] = {"segment_reduce": _device_ms(seg, repeats),
                     "scatter_add": _device_ms(scat, repeats)}
    segs = [out[k]["segment_reduce"] for k in ("uniform", "powerlaw")]
    scats = [out[k]["scatter_add"] for k in ("uniform", "powerlaw")]
    out["segment_reduce_variation"] = abs(segs[0] - segs[1]) / min(segs)
    out["scatter_add_variation"] = abs(scats[0] - scats[1]) / min(scats)
    return out
