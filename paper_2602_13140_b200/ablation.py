"""Materialising SchNet schedules on the GPU — the PipelineMode ablations
(reference flash.py:310-370, reference.py:100-209) and the paper's CGSchNet
baseline on the same hardware.

With fused=False the reference stacks every edge tensor (basis [E,Dr],
filter hidden [E,Fh], filters [E,D], gathered sources and messages [E,D])
in memory and aggregates either with an atomic scatter-add (segred=False,
the CGSchNet schedule) or with a CSR segmented reduction (segred=True).
This module runs exactly that on the GPU: cuBLAS GEMMs over the stacked
edge tensors, `index_add_` atomics or `fcg_segment_reduce`, and forces by
reverse-mode autodiff (F = -dE/dr), as CGSchNet does.  It is the ablation
arm and the same-GPU baseline, not the product path: the fused tcgen05
kernels of libfcg.so (PipelineMode() default) are.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from .engine import _torch
from .schnet import TrafficReport, traffic_report

LN2 = math.log(2.0)


def _layers(net):
    return net if isinstance(net, tuple) else net.layers


class TorchModel:
    """Device copy of ModelParams / QuantizedParams for the materialising
    schedule, in the compute dtype (fp32, or fp64 for fp64 inputs)."""

    def __init__(self, params, dtype, device="cuda"):
        torch = _torch()
        self.torch = torch
        self.dtype = dtype
        cfg = params.config
        self.cutoff = float(cfg.cutoff)
        t = lambda a: torch.as_tensor(np.asarray(a)).to(device=device, dtype=dtype)  # noqa: E731
        self.centers = t(np.asarray(params.rbf.centers, np.float64).astype(
            np.float32 if dtype == torch.float32 else np.float64))
        self.gamma = float(np.float32(params.rbf.gamma)) if dtype == torch.float32 \
            else float(params.rbf.gamma)
        self.embedding = t(params.embedding)
        self.quant = not isinstance(params.readout, tuple)

        def lin(layer):
            if isinstance(layer, tuple):
                return {"w": t(layer[0]), "b": t(layer[1]), "q": False}
            # quantize.py:55-71: fp16 inputs against scale * fp32(w16), fp32 bias
            return {"w": t(layer.dequant()), "b": t(layer.bias), "q": True}

        self.blocks = [dict(pre=lin(bp.pre_linear),
                            filt=[lin(x) for x in _layers(bp.filter_mlp)],
                            post=[lin(x) for x in _layers(bp.post_mlp)]) for bp in params.blocks]
        self.readout = [lin(x) for x in _layers(params.readout)]

    # model.py:93-100
    def ssp(self, x):
        torch = self.torch
        return torch.clamp_min(x, 0) + torch.log1p(torch.exp(-torch.abs(x))) - LN2

    def linear(self, layer, x):
        if layer["q"]:  # straight-through: the reference backward ignores the rounding
            x = x + (x.to(self.torch.float16).to(x.dtype) - x).detach()
        return x @ layer["w"].T + layer["b"]

    def mlp(self, net, x):
        for i, layer in enumerate(net):
            x = self.linear(layer, x)
            if i < len(net) - 1:
                x = self.ssp(x)
        return x


class _SegmentSum:
    """CSR segment sum with libfcg's contention-free kernel in the forward
    (flash.py:109-135) and a gather in the backward."""

    @staticmethod
    def make():
        torch = _torch()

        class Fn(torch.autograd.Function):
            @staticmethod
            def forward(ctx, values, ptr64, own):
                nseg = ptr64.numel() - 1
                k = values.shape[1]
                out = torch.empty(nseg, k, dtype=values.dtype, device=values.device)
                lib = _lib.load()
                fn = lib.fcg_segment_reduce_f64 if values.dtype == torch.float64 \
                    else lib.fcg_segment_reduce
                v = values.contiguous()
                wb = lib.fcg_segment_reduce_workspace_bytes(v.shape[0], k, nseg)
                ws = torch.empty(int(wb), dtype=torch.uint8, device=values.device)
                _lib.check(fn(_lib.vp(v), v.shape[0], k, _lib.vp(ptr64), nseg, _lib.vp(out),
                              _lib.vp(ws), wb,
                              C.c_void_p(torch.cuda.current_stream().cuda_stream)),
                           "fcg_segment_reduce")
                ctx.save_for_backward(own)
                return out

            @staticmethod
            def backward(ctx, g):
                (own,) = ctx.saved_tensors
                return g[own], None, None

        return Fn


_SEG = None


def materialized_energy_forces(model: TorchModel, pos, types, ptr, nbr, own, R: int, N: int,
                               segred: bool):
    """Energy per replica, per-atom energies and forces of a batch of R
    replicas ([R*N, 3] positions, block-diagonal CSR with edges grouped by
    destination: own = dst, nbr = src), materialising schedule."""
    global _SEG
    torch = model.torch
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False  # fp32 means fp32 here
    try:
        pos = pos.detach().to(model.dtype).requires_grad_(True)
        own_l, nbr_l = own.long(), nbr.long()
        # edge geometry (flash.py:219-223; _safe_inv at d <= TINY_DISTANCE)
        u = pos[own_l] - pos[nbr_l]
        s = (u[:, 0] * u[:, 0] + u[:, 1] * u[:, 1]) + u[:, 2] * u[:, 2]
        live = s > 1e-24
        d = torch.where(live, torch.sqrt(torch.where(live, s, torch.ones_like(s))),
                        torch.zeros_like(s))
        c = torch.where(d < model.cutoff,
                        0.5 * (torch.cos(math.pi * d / model.cutoff) + 1.0), torch.zeros_like(d))
        delta = d[:, None] - model.centers[None, :]
        basis = torch.exp(-model.gamma * delta * delta) * c[:, None]  # [E, Dr]
        types = types.long()
        if types.numel() == N and R > 1:  # per-bead types shared by the replicas
            types = types.repeat(R)
        X = model.embedding[types]
        if segred and _SEG is None:
            _SEG = _SegmentSum.make()
        ptr64 = ptr.long()
        for blk in model.blocks:
            P = model.linear(blk["pre"], X)
            W = model.mlp(blk["filt"], basis)           # [E, D] filters
            M = P[nbr_l] * W                           # [E, D] messages
            if segred:
                H = _SEG.apply(M, ptr64, own_l)
            else:  # CGSchNet: atomic scatter-add
                H = torch.zeros(X.shape[0], M.shape[1], dtype=M.dtype,
                                device=M.device).index_add_(0, own_l, M)
            X = X + model.mlp(blk["post"], H)
        per_atom = model.mlp(model.readout, X)[:, 0]
        energy = per_atom.reshape(R, N).sum(dim=1)
        (grad,) = torch.autograd.grad(energy.sum(), pos)
        return energy.detach(), per_atom.detach(), -grad
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32


def compare_on_engine(eng, params, reps: int = 5) -> dict:
    """Device time and peak memory of one energy+forces evaluation of the
    engine's replica batch with the fused kernels (segment sums, and the
    fused-scatter ablation with atomics: fcg_energy_forces_sched) and with
    the materialising schedules (scatter = CGSchNet, segmented), on the
    same positions and CSR.  CUDA events around each call; the materialising
    path's peak is measured above the memory already allocated."""
    torch = _torch()
    R, N = eng.R, eng.N
    c = eng.csr
    pos = eng.pos.reshape(R * N, 3)
    stream = torch.cuda.current_stream()
    L = _lib.load()
    ef = L.fcg_ef_workspace_bytes(C.byref(eng.model.desc), R, N, c.cap_e)
    ws = torch.empty(int(ef), dtype=torch.uint8, device=pos.device)
    per_atom = torch.empty(R * N, dtype=torch.float32, device=pos.device)
    energy = torch.empty(R, dtype=torch.float32, device=pos.device)
    forces = torch.empty(R * N, 3, dtype=torch.float32, device=pos.device)
    v = _lib.vp

    def flash(schedule=_lib.FCG_SCHED_SEGRED):
        return lambda: _lib.check(L.fcg_energy_forces_sched(
            C.byref(eng.model.desc), v(pos), v(eng.types), R, N, v(c.ptr), v(c.nbr), v(c.rev),
            v(c.own), c.cap_e, v(per_atom), v(energy), v(forces), v(ws), ef, schedule,
            C.c_void_p(stream.cuda_stream)), "fcg_energy_forces")

    model = TorchModel(params, torch.float32)
    E = int(c.ptr[-1].item())
    nbr, own = c.nbr[:E], c.own[:E]

    def mat(segred):
        return lambda: materialized_energy_forces(model, pos, eng.types, c.ptr, nbr, own, R, N,
                                                  segred)

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(reps):
            fn()
        t1.record()
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / reps, torch.cuda.max_memory_allocated() - base

    f_ms, f_mem = timed(flash())
    fs_ms, fs_mem = timed(flash(_lib.FCG_SCHED_SCATTER))
    s_ms, s_mem = timed(mat(False))
    g_ms, g_mem = timed(mat(True))
    return {"what": "one energy+forces evaluation of the replica batch, same positions and CSR",
            "replicas": R, "edges": int(c.ptr[-1].item()),
            "fused_ms": f_ms, "fused_scatter_ms": fs_ms,
            "materialized_scatter_ms": s_ms, "materialized_segred_ms": g_ms,
            "speedup_vs_fused_scatter": fs_ms / f_ms,
            "speedup_vs_scatter": s_ms / f_ms, "speedup_vs_segred": g_ms / f_ms,
            "extra_peak_bytes": {"fused": int(f_mem), "materialized_scatter": int(s_mem),
                                 "materialized_segred": int(g_mem)}}


class MaterializedReplicaForces:
    """force_fn(positions[R,N,3], step) -> (forces, {"potential", "prior"})
    with the materialising schedule (the reference's _ReplicaForces under a
    fused=False backend, md.py:231-273): device neighbour build, GPU
    materialised model forces, device harmonic prior."""

    def __init__(self, params, types, prior, config, segred: bool):
        from .prior import DevicePrior
        torch = _torch()
        self.torch, self.params, self.config, self.segred = torch, params, config, segred
        self.types = torch.as_tensor(np.asarray(types).astype(np.int64)).cuda()
        self.N = int(np.asarray(types).size)
        self.prior = DevicePrior(prior, self.N)
        self.model = TorchModel(params, torch.float32)
        self.edge_counts = []
        self.mode = config.backend
        self.traffic = TrafficReport()
        self._csr = None

    def __call__(self, positions, step):
        from .csr import device_csr
        torch = self.torch
        pos = np.asarray(positions, np.float32)
        R, N = pos.shape[0], pos.shape[1]
        if self._csr is None or step % max(self.config.neighbor_stride, 1) == 0:  # md.py:245
            p, nbr, _rev, own = device_csr(pos, self.model.cutoff)
            self._csr = tuple(torch.as_tensor(a).cuda() for a in (p, nbr, own))
            counts = p[N::N] - p[0:-1:N][:R]
            self._counts = [int(x) for x in counts]
        self.edge_counts.extend(self._counts)
        cfg = self.params.config
        for e in self._counts:   # md.py:267-268: every evaluation's modelled traffic
            self.traffic.merge(traffic_report(self.mode, N, e, cfg.hidden_dim, cfg.rbf_dim,
                                              len(self.params.blocks), 4))
        ptr, nbr, own = self._csr
        dpos = torch.as_tensor(pos).cuda()
        e, _pa, f = materialized_energy_forces(self.model, dpos.reshape(R * N, 3), self.types,
                                               ptr, nbr, own, R, N, self.segred)
        e_prior = torch.empty(R, device="cuda")
        f_prior = torch.empty(R, N, 3, device="cuda")
        _lib.check(_lib.load().fcg_prior_forces(C.byref(self.prior.desc), _lib.vp(dpos), R, N,
                                                _lib.vp(e_prior), _lib.vp(f_prior),
                                                C.c_void_p(torch.cuda.current_stream().cuda_stream)),
                   "fcg_prior_forces")
        forces = (f.reshape(R, N, 3).float() + f_prior).cpu().numpy()
        return forces, {"potential": e.double().cpu().numpy(),
                        "prior": e_prior.double().cpu().numpy()}
