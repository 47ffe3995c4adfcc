"""Model configuration and parameters, mirroring flashcg.model.

Host-side only: the types and the seeded initialiser are what a caller of
the reference constructs (model.py:164-459 of the reference); the compute
(basis, filter MLPs, node MLPs and their backward) runs in libfcg.so.
`init_params` reproduces the reference's draws bit for bit (pinned by
tests/test_host.py (hash-pinned: test_init_params_bit_identical, test_generate_system_bit_identical, test_quantize_model_bit_identical) against fixtures generated from the reference).
`DeviceModel` packs a parameter set into zero-padded device tensors plus
the `fcg_model` descriptor the C ABI consumes.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

LN2 = math.log(2.0)

DEFAULT_HIDDEN_DIM = 128
DEFAULT_RBF_DIM = 64
DEFAULT_NUM_BLOCKS = 3
DEFAULT_CUTOFF = 1.5  # nm
DEFAULT_NUM_ATOM_TYPES = 32
DEFAULT_FILTER_HIDDEN = 128
DEFAULT_READOUT_HIDDEN = 64


class ConfigError(ValueError):
    """Invalid model configuration or mismatched shapes (reference model.py:28)."""


@dataclass(frozen=True)
class ModelConfig:
    hidden_dim: int = DEFAULT_HIDDEN_DIM
    rbf_dim: int = DEFAULT_RBF_DIM
    num_blocks: int = DEFAULT_NUM_BLOCKS
    cutoff: float = DEFAULT_CUTOFF
    num_atom_types: int = DEFAULT_NUM_ATOM_TYPES
    filter_hidden_dim: int = DEFAULT_FILTER_HIDDEN
    readout_hidden_dim: int = DEFAULT_READOUT_HIDDEN

    def __post_init__(self):
        ints = ("hidden_dim", "rbf_dim", "num_blocks", "num_atom_types",
                "filter_hidden_dim", "readout_hidden_dim")
        bad = [k for k in ints if int(getattr(self, k)) < 1]
        if bad:
            raise ConfigError(f"{bad[0]} must be >= 1, got {getattr(self, bad[0])}")
        if not self.cutoff > 0:
            raise ConfigError(f"cutoff must be > 0, got {self.cutoff}")


@dataclass(frozen=True)
class RbfSpec:
    """Gaussian centres on [0, cutoff] with one shared width (model.py:51-90)."""

    centers: np.ndarray
    gamma: float
    cutoff: float

    def __post_init__(self):
        c = np.asarray(self.centers, dtype=np.float64)
        if c.ndim != 1 or c.size == 0:
            raise ConfigError("centers must be a non-empty 1-d array")
        if not self.gamma > 0:
            raise ConfigError(f"gamma must be > 0, got {self.gamma}")
        if c.size > 1 and (np.any(np.diff(c) <= 0) or c[0] != 0.0
                           or not np.isclose(c[-1], self.cutoff)):
            raise ConfigError("centers must increase strictly over [0, cutoff]")

    @property
    def dim(self) -> int:
        return int(np.asarray(self.centers).size)

    @classmethod
    def uniform(cls, rbf_dim: int, cutoff: float) -> "RbfSpec":
        if rbf_dim < 2:
            return cls(centers=np.zeros(1), gamma=1.0 / (2.0 * cutoff * cutoff),
                       cutoff=float(cutoff))
        delta = cutoff / (rbf_dim - 1)
        return cls(centers=np.linspace(0.0, cutoff, rbf_dim),
                   gamma=1.0 / (2.0 * delta * delta), cutoff=float(cutoff))

    @classmethod
    def for_config(cls, config: ModelConfig) -> "RbfSpec":
        return cls.uniform(config.rbf_dim, config.cutoff)


@dataclass(frozen=True)
class BlockParams:
    pre_linear: tuple   # (W[D,D], b[D])
    filter_mlp: tuple   # ((W[Fh,Dr], b), (W[D,Fh], b))
    post_mlp: tuple     # ((W[D,D], b), (W[D,D], b))


@dataclass(frozen=True)
class ModelParams:
    config: ModelConfig
    embedding: np.ndarray
    blocks: tuple
    readout: tuple      # ((W[Rh,D], b), (W[1,Rh], b))
    rbf: RbfSpec = field(default=None)

    def __post_init__(self):
        if self.rbf is None:
            object.__setattr__(self, "rbf", RbfSpec.for_config(self.config))

    @property
    def dtype(self):
        return self.embedding.dtype

    def astype(self, dtype) -> "ModelParams":
        def cast(layers):
            return tuple((w.astype(dtype), b.astype(dtype)) for w, b in layers)
        return ModelParams(
            config=self.config, embedding=self.embedding.astype(dtype),
            blocks=tuple(BlockParams(pre_linear=cast([bp.pre_linear])[0],
                                     filter_mlp=cast(bp.filter_mlp),
                                     post_mlp=cast(bp.post_mlp)) for bp in self.blocks),
            readout=cast(self.readout), rbf=self.rbf)

    def named_tensors(self):
        out = [("embedding", self.embedding)]
        for t, bp in enumerate(self.blocks):
            out += [(f"block{t}.pre.W", bp.pre_linear[0]), (f"block{t}.pre.b", bp.pre_linear[1])]
            for kind, layers in (("filter", bp.filter_mlp), ("post", bp.post_mlp)):
                for j, (w, b) in enumerate(layers):
                    out += [(f"block{t}.{kind}{j}.W", w), (f"block{t}.{kind}{j}.b", b)]
        for j, (w, b) in enumerate(self.readout):
            out += [(f"readout{j}.W", w), (f"readout{j}.b", b)]
        return out


def init_params(config: ModelConfig, seed: int) -> ModelParams:
    """Glorot-uniform weights drawn in float64 from default_rng(seed), zero
    biases, stored float32 — the reference's draw order (model.py:292-327):
    embedding, then per block pre, filter0, filter1, post0, post1, then the
    two readout layers."""
    rng = np.random.default_rng(seed)
    d, dr = config.hidden_dim, config.rbf_dim
    fh, rh = config.filter_hidden_dim, config.readout_hidden_dim

    def layer(n_out, n_in):
        bound = math.sqrt(6.0 / (n_in + n_out))
        return rng.uniform(-bound, bound, size=(n_out, n_in)), np.zeros(n_out)

    emb = rng.uniform(-1.0, 1.0, size=(config.num_atom_types, d)) / math.sqrt(d)
    blocks = []
    for _ in range(config.num_blocks):
        pre = layer(d, d)
        filt = (layer(fh, dr), layer(d, fh))
        post = (layer(d, d), layer(d, d))
        blocks.append(BlockParams(pre_linear=pre, filter_mlp=filt, post_mlp=post))
    readout = (layer(rh, d), layer(1, rh))
    return ModelParams(config=config, embedding=emb, blocks=tuple(blocks),
                       readout=readout).astype(np.float32)


# ---------------------------------------------------------------------------
# device packing

def _check_widths(cfg: ModelConfig):
    lim = {"hidden_dim": _lib.FCG_D, "filter_hidden_dim": _lib.FCG_D,
           "rbf_dim": _lib.FCG_DR, "readout_hidden_dim": _lib.FCG_RH,
           "num_blocks": _lib.FCG_MAX_BLOCKS}
    for k, v in lim.items():
        if getattr(cfg, k) > v:
            raise ConfigError(f"{k}={getattr(cfg, k)} exceeds the compiled width {v} of libfcg")


def _pad(a, shape):
    out = np.zeros(shape, dtype=np.float32)
    a = np.asarray(a, dtype=np.float32)
    out[tuple(slice(0, s) for s in a.shape)] = a
    return out


def core_matrix_image(w: np.ndarray) -> np.ndarray:
    """(out, in) matrix -> flat canonical no-swizzle core-matrix order used by
    the tcgen05 descriptors: 8x8 blocks of 128 bytes, row-block major."""
    R, Cc = w.shape
    assert R % 8 == 0 and Cc % 8 == 0
    return np.ascontiguousarray(w.reshape(R // 8, 8, Cc // 8, 8).transpose(0, 2, 1, 3)).reshape(-1)


def tc_image(w: np.ndarray, quantized_f16: np.ndarray | None = None):
    """fp16 (hi, lo) operand image of a padded (out, in) weight matrix and its
    power-of-two prescale exponent.  fp32 weights: W*2^e = hi + lo (~22-bit
    split, max|W*2^e| <= 2^15).  W16 weights: hi = stored fp16, lo = 0."""
    if quantized_f16 is not None:
        hi = quantized_f16.astype(np.float16)
        return np.concatenate([core_matrix_image(hi), np.zeros(hi.size, np.float16)]), 0
    w = np.asarray(w, np.float32)
    amax = float(np.max(np.abs(w))) if w.size else 0.0
    e = 14 - int(np.floor(np.log2(amax))) if amax > 0 else 0
    ws = (w.astype(np.float64) * 2.0 ** e).astype(np.float32)
    hi = ws.astype(np.float16)
    lo = (ws - hi.astype(np.float32)).astype(np.float16)
    return np.concatenate([core_matrix_image(hi), core_matrix_image(lo)]), e


def _pow2_exp(bound: float) -> int:
    """e with bound * 2^e in [2^14, 2^15): the fp16 hi/lo operand split of a
    value |x| <= bound then never overflows and keeps ~22 bits (absolute
    error <= bound * 2^-39 below that)."""
    return 14 - int(np.floor(np.log2(bound))) if bound > 0 else 0


def _dgrid_basis(centers, gamma: float, cutoff: float, n: int = 30001):
    """Basis rows b(d) (model.py:123-133) and their derivatives on a grid of
    d over [0, cutoff], 2,000x finer than the basis width."""
    d = np.linspace(0.0, float(cutoff), n)
    delta = d[:, None] - np.asarray(centers, np.float64)[None, :]
    env = 0.5 * (np.cos(np.pi * d / cutoff) + 1.0)
    denv = -0.5 * np.pi / cutoff * np.sin(np.pi * d / cutoff)
    g = np.exp(-gamma * delta * delta)
    return g * env[:, None], g * (-2.0 * gamma * delta * env[:, None] + denv[:, None])


def edge_h_exp(w0: np.ndarray, b0: np.ndarray, centers=None, gamma: float = 0.0,
               cutoff: float = 0.0) -> int:
    """Static scale of h = ssp(W0 b(d) + b0) in the edge kernels.  z0 depends
    on the edge only through d, so max |h| over d in [0, cutoff] (a grid
    2,000x finer than the basis width, 5% margin; the split tolerates 2x
    more before fp16 overflows) bounds it tightly — about 30x below the
    algebraic bound sum_k |W0[c,k]| + |b0[c]| (0 <= b <= 1), which the hi/lo
    split would otherwise spend as 5 bits of precision.  Without the basis
    parameters the algebraic bound is used."""
    w0 = np.asarray(w0, np.float64)
    b0 = np.asarray(b0, np.float64)
    if centers is None:
        bz = float(np.max(np.sum(np.abs(w0), axis=1) + np.abs(b0)))
        return _pow2_exp(max(bz, math.log(2.0)) * 1.001)
    b, _ = _dgrid_basis(centers, gamma, cutoff)
    z = b @ w0.T + b0
    h = np.maximum(z, 0) + np.log1p(np.exp(-np.abs(z))) - math.log(2.0)
    return _pow2_exp(float(np.max(np.abs(h))) * 1.05)


def edge_db_exp(gamma: float, cutoff: float) -> int:
    """Static scale of the basis derivative db_k = g_k (-2 gamma delta_k C +
    C') (model.py:136-157): |2 gamma delta exp(-gamma delta^2)| <=
    sqrt(2 gamma / e), 0 <= C <= 1, |C'| <= pi / (2 r_cut)."""
    return _pow2_exp((math.sqrt(2.0 * gamma / math.e) + math.pi / (2.0 * cutoff)) * 1.001)


def edge_v_exp(w0: np.ndarray, centers: np.ndarray, gamma: float, cutoff: float) -> int:
    """Static scale of v = ssp'(z0) * (W0 db) in the forward-mode backward
    edge kernel (csrc/edge_tc.cu, k_edge_bwd_fm): 0 < ssp' < 1, so |v[c]| <=
    max over d of sum_k |W0[c,k]| |db_k(d)| (model.py:136-157), evaluated on
    a grid 2,000x finer than the basis width (the function moves < 0.5%
    between points; 5% margin, and the split tolerates 2x before fp16
    overflows)."""
    _, db = _dgrid_basis(centers, gamma, cutoff)
    bound = float(np.max(np.abs(db) @ np.abs(w0.astype(np.float64)).T))
    return _pow2_exp(bound * 1.05)


def _is_quantized(params) -> bool:
    return not isinstance(params.readout, tuple)


class DeviceModel:
    """Zero-padded device copy of ModelParams / QuantizedParams + descriptor.

    Weights are uploaded once per process and shared read-only by all
    replicas; the descriptor holds raw device pointers into
    the tensors kept alive here.
    """

    def __init__(self, params, device="cuda"):
        import torch

        cfg = params.config
        _check_widths(cfg)
        self.config = cfg
        self.quantized = _is_quantized(params)
        self._keep = []
        D, DR, RH = _lib.FCG_D, _lib.FCG_DR, _lib.FCG_RH

        def dev(a, dtype=torch.float32):
            t = torch.as_tensor(np.ascontiguousarray(a)).to(device=device, dtype=dtype)
            self._keep.append(t)
            return t

        def dense(lin):
            """fp32 (out,in) matrix the backward uses: W, or dequant() for W16."""
            if isinstance(lin, tuple):
                return np.asarray(lin[0], np.float32), np.asarray(lin[1], np.float32)
            return lin.dequant().astype(np.float32), np.asarray(lin.bias, np.float32)

        def layers_of(net):
            return net if isinstance(net, tuple) else net.layers

        def image_of(lin, shape):
            if isinstance(lin, tuple):
                return tc_image(_pad(lin[0], shape))
            q = np.zeros(shape, np.float16)
            q[:lin.weight.shape[0], :lin.weight.shape[1]] = lin.weight
            return tc_image(None, q)

        m = _lib.FcgModel()
        m.format = _lib.FCG_FMT_W16 if self.quantized else _lib.FCG_FMT_FP32
        m.num_blocks = len(params.blocks)
        m.num_types = int(params.embedding.shape[0])
        m.cutoff = float(np.float32(cfg.cutoff))
        m.gamma = float(np.float32(params.rbf.gamma))
        m.centers = _lib.fptr(dev(_pad(np.asarray(params.rbf.centers).astype(np.float32), (DR,))))
        m.embedding = _lib.fptr(dev(_pad(params.embedding, (m.num_types, D))))

        def put(blk, name, lin, shape_out, shape_in, quant_src=None):
            w, b = dense(lin)
            wp = _pad(w, (shape_out, shape_in))
            setattr(blk, f"{name}_w", _lib.fptr(dev(wp)))
            setattr(blk, f"{name}_wt", _lib.fptr(dev(np.ascontiguousarray(wp.T))))
            setattr(blk, f"{name}_b", _lib.fptr(dev(_pad(b, (shape_out,)))))
            if not isinstance(lin, tuple):
                w16 = np.zeros((shape_out, shape_in), dtype=np.float16)
                w16[:lin.weight.shape[0], :lin.weight.shape[1]] = lin.weight
                setattr(blk, f"{name}_h", _lib.u16ptr(dev(w16.view(np.int16), torch.int16)))
                sc = np.ones(shape_out, np.float32)
                sc[:lin.scale.shape[0]] = lin.scale
                setattr(blk, f"{name}_s", _lib.fptr(dev(sc)))

        for t, bp in enumerate(params.blocks):
            blk = m.blocks[t]
            f0, f1 = layers_of(bp.filter_mlp)
            p0, p1 = layers_of(bp.post_mlp)
            put(blk, "pre", bp.pre_linear, D, D)
            put(blk, "f0", f0, D, DR)
            put(blk, "f1", f1, D, D)
            put(blk, "p0", p0, D, D)
            put(blk, "p1", p1, D, D)
            for name, lin, shape in (("f0", f0, (D, DR)), ("f1", f1, (D, D)),
                                     ("pre", bp.pre_linear, (D, D)), ("p0", p0, (D, D)),
                                     ("p1", p1, (D, D))):
                img, e = image_of(lin, shape)
                setattr(blk, f"{name}_img", _lib.u16ptr(dev(img.view(np.int16), torch.int16)))
                setattr(blk, f"{name}_exp", e)
            w0, b0 = dense(f0)
            blk.f_hexp = edge_h_exp(w0, b0, params.rbf.centers, float(params.rbf.gamma),
                                    float(cfg.cutoff))
            blk.f_dbexp = edge_db_exp(float(np.float32(params.rbf.gamma)), float(cfg.cutoff))
            blk.f1_qmax = 1.0 if isinstance(f1, tuple) else float(np.max(f1.scale))
            blk.f_vexp = edge_v_exp(w0, params.rbf.centers, float(params.rbf.gamma),
                                    float(cfg.cutoff))

        # block 0's pre-linear of every embedding row (fcg_model.pre0_table):
        # X_0 = embedding[types] is position-independent, so P_0 is a table
        # gathered per step instead of a GEMM (evaluated in fp64 from the
        # reference's operands, W16: fp16-rounded inputs and dequantised
        # weights as quantize.py:68-71, then rounded to fp32)
        if params.blocks:
            lin0 = params.blocks[0].pre_linear
            emb = np.asarray(params.embedding, np.float32)
            if isinstance(lin0, tuple):
                x, (w, b) = emb.astype(np.float64), (np.asarray(lin0[0]), np.asarray(lin0[1]))
            else:
                x = emb.astype(np.float16).astype(np.float64)
                w, b = lin0.dequant(), np.asarray(lin0.bias)
            tab = (x @ np.asarray(w, np.float64).T + np.asarray(b, np.float64)).astype(np.float32)
            m.pre0_table = _lib.fptr(dev(_pad(tab, (m.num_types, D))))
            m.pre0_amax = float(np.max(np.abs(tab))) if tab.size else 0.0

        r0, r1 = layers_of(params.readout)
        img, e = image_of(r0, (RH, D))
        m.r0_img = _lib.u16ptr(dev(img.view(np.int16), torch.int16))
        m.r0_exp = e
        if not isinstance(r0, tuple):
            sc = np.ones(RH, np.float32)
            sc[:r0.scale.shape[0]] = r0.scale
            m.r0_s = _lib.fptr(dev(sc))
        w0, b0 = dense(r0)
        w0p = _pad(w0, (RH, D))
        m.r0_w = _lib.fptr(dev(w0p))
        m.r0_wt = _lib.fptr(dev(np.ascontiguousarray(w0p.T)))
        m.r0_b = _lib.fptr(dev(_pad(b0, (RH,))))
        w1, b1 = dense(r1)
        m.r1_w = _lib.fptr(dev(_pad(w1.reshape(-1), (RH,))))
        m.r1_b = float(np.float32(b1.reshape(-1)[0]))
        self.desc = m
