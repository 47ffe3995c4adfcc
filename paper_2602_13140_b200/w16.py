"""Channel-wise 16-bit weights: the QuantizedLinear / QuantizedMlp /
QuantizedParams containers of the reference (quantize.py:55-123) and the
offline calibration `quantize_model` (quantize.py:126-299), run on the host.

The GPU consumes these through DeviceModel: fp16 stored weights plus fp32
per-output-channel scales for the forward, and the fp32 dequantised matrix
scale[:,None]*fp32(w16) for the backward.  Calibration is a one-off CPU
step; it reproduces the reference's choice of scales bit for bit (pinned by
tests/test_host.py (hash-pinned: test_init_params_bit_identical, test_generate_system_bit_identical, test_quantize_model_bit_identical)) so the C3 benchmark weights are the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .modelparams import BlockParams, ModelConfig, ModelParams, RbfSpec

SCALE_GRID_SIZE = 33
SCALE_GRID_SPAN = 8.0
MIN_CALIBRATION_SAMPLES = 32
_GRID = np.geomspace(1.0 / SCALE_GRID_SPAN, SCALE_GRID_SPAN, SCALE_GRID_SIZE)


@dataclass(frozen=True)
class QuantizedLinear:
    weight: np.ndarray  # float16 (out, in), original / scale
    scale: np.ndarray   # float32 (out,), > 0
    bias: np.ndarray    # float32 (out,)

    def __post_init__(self):
        if not np.all(np.isfinite(self.scale)) or np.any(self.scale <= 0):
            raise ValueError("scales must be finite and strictly positive")

    def dequant(self) -> np.ndarray:
        return self.scale[:, None] * self.weight.astype(np.float32)


@dataclass(frozen=True)
class QuantizedMlp:
    layers: tuple


@dataclass(frozen=True)
class QuantizedParams:
    config: ModelConfig
    embedding: np.ndarray
    blocks: tuple
    readout: QuantizedMlp
    rbf: RbfSpec

    @property
    def dtype(self):
        return self.embedding.dtype


# ---------------------------------------------------------------------------
# calibration (host, float64)

def _ssp64(x):
    return np.maximum(x, 0) + np.log1p(np.exp(-np.abs(x))) - np.log(2.0)


def _basis64(d, rbf: RbfSpec):
    mu = np.asarray(rbf.centers, dtype=np.float64)
    dl = d[..., None] - mu
    env = np.where(d < rbf.cutoff, 0.5 * (np.cos(np.pi * d / rbf.cutoff) + 1.0), 0.0)
    return np.exp(-d.dtype.type(rbf.gamma) * dl * dl) * env[..., None]


def _host_errors(w: np.ndarray, cand: np.ndarray, gram: np.ndarray) -> np.ndarray:
    """err[r][c] = dw' G dw of every (row, candidate) pair, with the
    reference's own numpy operations (quantize.py:150-170)."""
    q = (w[:, None, :] / cand[:, :, None]).astype(np.float16)
    dw = q.astype(np.float64) * cand[:, :, None] - w[:, None, :]
    dw = np.where(np.isfinite(dw), dw, 1e30)
    flat = dw.reshape(-1, w.shape[1])
    return np.einsum("si,si->s", flat @ gram, flat).reshape(cand.shape)


# relative gap below which the GPU's best two candidates count as a tie (the
# device sums in another order than numpy's BLAS, ~1e-15 relative apart)
_TIE_RTOL = 1e-9


def _device_errors(w: np.ndarray, cand: np.ndarray, gram: np.ndarray, device) -> np.ndarray:
    """The same scores from libfcg's fcg_calib_errors (csrc/calib.cu).  When
    any row's best two candidates are within _TIE_RTOL, the layer is scored
    on the host instead, so argmin — the stored scale — is the reference's."""
    import ctypes as C

    from . import _lib
    from .engine import _torch

    torch = _torch()
    lib = _lib.load()
    dev = torch.device(device)
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.float64)).to(dev)  # noqa: E731
    dw_, dc, dg = t(w), t(cand), t(gram)
    err = torch.empty(cand.shape, dtype=torch.float64, device=dev)
    v = _lib.vp
    _lib.check(lib.fcg_calib_errors(v(dw_), w.shape[0], w.shape[1], v(dc), cand.shape[1], v(dg),
                                    v(err), C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)),
               "fcg_calib_errors")
    e = err.cpu().numpy()
    part = np.sort(e, axis=1)[:, :2] if e.shape[1] > 1 else np.concatenate([e, e + 1.0], axis=1)
    if np.any(part[:, 1] - part[:, 0] <= _TIE_RTOL * np.abs(part[:, 0])):
        return _host_errors(w, cand, gram)
    return e


def _calibrated(w: np.ndarray, b: np.ndarray, samples: np.ndarray,
                device=None) -> QuantizedLinear:
    """Per-row scale minimising dw' G dw over a geometric grid around the row
    absmax, the tensor-wide grid and 1.0 (quantize.py:126-178); the scores
    on the GPU when `device` is given."""
    if samples.ndim != 2 or samples.shape[0] < MIN_CALIBRATION_SAMPLES:
        raise ValueError(f"calibration needs at least {MIN_CALIBRATION_SAMPLES} samples")
    w = np.asarray(w, dtype=np.float64)
    s64 = samples.astype(np.float64)
    gram = s64.T @ s64
    amax = np.abs(w).max(axis=1)
    dead = amax == 0.0
    seeds = np.where(dead, 1.0, amax)
    tensor_grid = (float(np.abs(w).max()) or 1.0) * _GRID
    shared = np.concatenate([tensor_grid, [1.0]])
    cand = np.concatenate([seeds[:, None] * _GRID[None, :],
                           np.broadcast_to(shared, (w.shape[0], shared.size))], axis=1)
    cand = np.sort(cand, axis=1)
    if device is not None and w.shape[1] <= 256:
        err = _device_errors(w, cand, gram, device)
    else:
        err = _host_errors(w, cand, gram)
    scale = cand[np.arange(w.shape[0]), np.argmin(err, axis=1)]
    scale[dead] = 1.0
    stored = (w / scale[:, None]).astype(np.float16)
    stored[dead] = 0.0
    return QuantizedLinear(weight=stored, scale=scale.astype(np.float32),
                           bias=np.asarray(b, dtype=np.float32))


def _calibrated_mlp(layers, x: np.ndarray, device=None) -> QuantizedMlp:
    out, a = [], x
    for i, (w, b) in enumerate(layers):
        out.append(_calibrated(w, b, a, device))
        z = a @ np.asarray(w, dtype=np.float64).T + b
        if i < len(layers) - 1:
            a = _ssp64(z)
    return QuantizedMlp(tuple(out))


def _pairs64(pos: np.ndarray, r_cut: float):
    diff = pos[:, None, :] - pos[None, :, :]
    mask = np.einsum("ijk,ijk->ij", diff, diff) < r_cut * r_cut
    np.fill_diagonal(mask, False)
    dst, src = np.nonzero(mask)
    return src, dst


def _node_samples(params: ModelParams, seed: int, n_states: int = 4, n_beads: int = 48):
    """Block inputs recorded from fp64 forward passes on random boxes
    (quantize.py:224-260)."""
    rng = np.random.default_rng(seed)
    cfg = params.config
    box = 0.6 * cfg.cutoff * max(1.0, n_beads ** (1.0 / 3.0))
    p64 = params.astype(np.float64)
    T = len(p64.blocks)
    pre_in, post_in, ro_in = [[] for _ in range(T)], [[] for _ in range(T)], []
    for _ in range(n_states):
        pos = rng.uniform(0.0, box, size=(n_beads, 3))
        types = rng.integers(0, cfg.num_atom_types, size=n_beads)
        src, dst = _pairs64(pos, cfg.cutoff)
        u = pos[dst] - pos[src]
        d = np.sqrt(np.einsum("ij,ij->i", u, u))
        X = p64.embedding[types]
        for t, bp in enumerate(p64.blocks):
            pre_in[t].append(X)
            P = X @ bp.pre_linear[0].T + bp.pre_linear[1]
            a = _basis64(d, p64.rbf)
            for i, (w, b) in enumerate(bp.filter_mlp):
                a = a @ w.T + b
                if i < len(bp.filter_mlp) - 1:
                    a = _ssp64(a)
            H = np.zeros_like(X)
            np.add.at(H, dst, P[src] * a)
            post_in[t].append(H)
            h = H
            for i, (w, b) in enumerate(bp.post_mlp):
                h = h @ w.T + b
                if i < len(bp.post_mlp) - 1:
                    h = _ssp64(h)
            X = X + h
        ro_in.append(X)
    cat = lambda parts: np.concatenate(parts, axis=0)  # noqa: E731
    return [cat(p) for p in pre_in], [cat(p) for p in post_in], cat(ro_in)


def quantize_model(params: ModelParams, seed: int = 0, n_rbf_samples: int = 256,
                   device=None) -> QuantizedParams:
    """quantize.py:264-299.  device="cuda" scores the calibration candidates
    with fcg_calib_errors on the GPU (bit-identical result: near-ties are
    re-scored on the host); the default is the host computation."""
    rng = np.random.default_rng(seed)
    cfg = params.config
    rbf_in = _basis64(rng.uniform(0.0, cfg.cutoff, size=n_rbf_samples).astype(np.float64),
                      params.rbf)
    pre_in, post_in, ro_in = _node_samples(params, seed + 1)
    blocks = []
    for t, bp in enumerate(params.blocks):
        blocks.append(BlockParams(
            pre_linear=_calibrated(bp.pre_linear[0], bp.pre_linear[1], pre_in[t], device),
            filter_mlp=_calibrated_mlp(bp.filter_mlp, rbf_in, device),
            post_mlp=_calibrated_mlp(bp.post_mlp, post_in[t], device)))
    return QuantizedParams(config=cfg, embedding=params.embedding.astype(np.float32),
                           blocks=tuple(blocks),
                           readout=_calibrated_mlp(params.readout, ro_in, device),
                           rbf=params.rbf)
