"""Device-resident batched MD engine over libfcg.so.

One engine holds R replicas of one system on one GPU: parameters uploaded
once, state (positions, velocities, forces, step counter, status words),
the flattened CSR buffers, and one workspace.  A step is a single
fcg_md_step call (noise -> BAOA -> neighbour rebuild -> prior -> energy and
forces -> trailing half-kick), so K steps can be captured into one CUDA
graph and replayed with no host involvement; the host only reads state at
output strides.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from .modelparams import DeviceModel
from .prior import DevicePrior

KB = 0.00831446261815324  # kJ/(mol K), md.py:29


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2602_13140_b200 requires a CUDA device (no CPU fallback)")
    return torch


def md_params(dt_fs: float, temperature: float, friction: float, seed: int,
              rep_offset: int = 0, neighbor_stride: int = 1) -> _lib.FcgMdParams:
    """Coefficients as numpy 2 evaluates them in fp32 mode (md.py:158-169):
    Python-float expressions are computed in double, then rounded to fp32."""
    dt = dt_fs * 1.0e-3
    c1 = math.exp(-friction * dt)
    p = _lib.FcgMdParams()
    p.half_dt = float(np.float32(0.5 * dt))
    p.c1 = float(np.float32(c1))
    p.c2_num = float(np.float32((1.0 - c1 * c1) * KB * temperature))
    p.seed = int(seed)
    p.rep_offset = int(rep_offset)
    p.neighbor_stride = int(max(neighbor_stride, 1))
    return p


class CsrBuffers:
    """Flattened CSR over R*N nodes (see include/fcg.h)."""

    def __init__(self, R: int, N: int, cap_e: int, device):
        torch = _torch()
        self.R, self.N, self.cap_e = R, N, int(cap_e)
        self.ptr = torch.zeros(R * N + 1, dtype=torch.int32, device=device)
        self.nbr = torch.zeros(self.cap_e + 1, dtype=torch.int32, device=device)
        self.rev = torch.zeros(self.cap_e + 1, dtype=torch.int32, device=device)
        self.own = torch.zeros(self.cap_e + 1, dtype=torch.int32, device=device)

    def slice_replica(self, r: int):
        """Reference-layout (src, dst, ptr, perm_src) of replica r as int64 numpy."""
        ptr = self.ptr.cpu().numpy().astype(np.int64)
        N = self.N
        lo, hi = ptr[r * N], ptr[(r + 1) * N]
        src = self.nbr[lo:hi].cpu().numpy().astype(np.int64) - r * N
        dst = self.own[lo:hi].cpu().numpy().astype(np.int64) - r * N
        rev = self.rev[lo:hi].cpu().numpy().astype(np.int64) - lo
        return src, dst, ptr[r * N:(r + 1) * N + 1] - lo, rev


def default_capacity(R: int, N: int) -> int:
    dense = R * N * (N - 1)
    return int(max(1, min(dense, R * N * 96)))


class MDEngine:
    def __init__(self, params, types, masses, prior, n_replicas: int, dt_fs=4.0,
                 temperature=300.0, friction=1.0, seed=0, neighbor_stride=1, rep_offset=0,
                 cap_e: int | None = None, device="cuda", schedule: int = _lib.FCG_SCHED_SEGRED):
        torch = _torch()
        self.torch = torch
        self.lib = _lib.load()
        self.device = torch.device(device)
        types = np.asarray(types)
        N = int(types.size)
        R = int(n_replicas)
        if np.any(types < 0) or np.any(types >= params.config.num_atom_types):
            raise ValueError("atom type out of range for the embedding table")
        self.R, self.N = R, N
        self.r_cut = float(params.config.cutoff)
        self.model = DeviceModel(params, self.device)
        self.prior = DevicePrior(prior, N, self.device)
        self.p = md_params(dt_fs, temperature, friction, seed, rep_offset, neighbor_stride)
        # aggregation schedule of the force evaluation: segment sums (the
        # product path) or the fused-scatter ablation (include/fcg.h)
        self.schedule = int(schedule)
        self.p.schedule = self.schedule
        self.mass = torch.as_tensor(np.asarray(masses, np.float64).astype(np.float32),
                                    device=self.device)
        self.masses64 = np.asarray(masses, np.float64)
        self.types = torch.as_tensor(types.astype(np.int32), device=self.device)
        f32 = dict(dtype=torch.float32, device=self.device)
        # positions and velocities are views of one buffer (and the two
        # per-replica energies of another), so host I/O of a step's state is
        # one copy per direction
        self.state = torch.zeros(2, R, N, 3, **f32)
        self.pos, self.vel = self.state[0], self.state[1]
        self.forces = torch.zeros(R, N, 3, **f32)
        self.energies = torch.zeros(2, R, **f32)
        self.potential, self.prior_e = self.energies[0], self.energies[1]
        self.step = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.status = torch.zeros(_lib.FCG_STATUS_WORDS, dtype=torch.int64, device=self.device)
        self._alloc(cap_e or default_capacity(R, N))
        self._graphs = {}

    # -- buffers ---------------------------------------------------------
    def _alloc(self, cap_e: int, keep: dict | None = None):
        torch = self.torch
        self.csr = CsrBuffers(self.R, self.N, cap_e, self.device)
        if keep is not None:  # restore a saved CSR (see save_csr) into the new buffers
            self.csr.ptr.copy_(keep["ptr"])
            for k in ("nbr", "rev", "own"):
                src = keep[k]
                getattr(self.csr, k)[:src.numel()].copy_(src)
        nbytes = self.lib.fcg_md_workspace_bytes(C.byref(self.model.desc), self.R, self.N,
                                                 self.csr.cap_e)
        # zero-filled: the noise ring's validity tag lives in this workspace,
        # and a recycled allocation must never carry a stale tag that matches
        self.ws = torch.zeros(int(nbytes), dtype=torch.uint8, device=self.device)
        self._graphs = {}

    @property
    def cap_e(self) -> int:
        return self.csr.cap_e

    def save_csr(self) -> dict:
        """Copy of the live CSR (needed to replay a chunk exactly when the
        neighbour list is only rebuilt every neighbor_stride steps)."""
        e = int(self.csr.ptr[-1].item())
        e = min(e, self.cap_e)
        return {"ptr": self.csr.ptr.clone(), "nbr": self.csr.nbr[:e].clone(),
                "rev": self.csr.rev[:e].clone(), "own": self.csr.own[:e].clone()}

    def stream(self):
        return C.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    # -- state -----------------------------------------------------------
    def load_state(self, positions, velocities, step: int):
        self.pos.copy_(self.torch.as_tensor(np.asarray(positions, np.float32)))
        self.vel.copy_(self.torch.as_tensor(np.asarray(velocities, np.float32)))
        self.step.fill_(int(step))

    def read_state(self):
        return (self.pos.cpu().numpy(), self.vel.cpu().numpy(), int(self.step.item()))

    # -- kernels ---------------------------------------------------------
    def _md_step(self):
        L, c, v = self.lib, self.csr, _lib.vp
        rc = L.fcg_md_step(C.byref(self.model.desc), C.byref(self.prior.desc), C.byref(self.p),
                           v(self.mass), v(self.types), self.R, self.N, self.r_cut, c.cap_e,
                           v(self.step), v(self.pos), v(self.vel), v(self.forces),
                           v(self.potential), v(self.prior_e), v(c.ptr), v(c.nbr), v(c.rev),
                           v(c.own), v(self.status), v(self.ws), self.ws.numel(), self.stream())
        _lib.check(rc, "fcg_md_step")

    def evaluate(self, rebuild: bool = True):
        """Forces of the current positions (the integrate() pre-loop force
        evaluation, md.py:195): neighbour build + prior + model, no kick.
        rebuild=False reuses the current CSR (neighbor_stride > 1,
        md.py:245-250)."""
        L, v = self.lib, _lib.vp
        torch = self.torch
        while rebuild:
            c = self.csr  # re-read: a regrow below replaces the buffers
            nb = L.fcg_nbr_workspace_bytes(self.R, self.N)
            ws_nb = torch.zeros(int(nb), dtype=torch.uint8, device=self.device)  # fcg.h contract
            _lib.check(L.fcg_nbr_build(v(self.pos), self.R, self.N, self.r_cut, c.cap_e, v(c.ptr),
                                       v(c.nbr), v(c.rev), v(c.own), v(self.status), v(ws_nb),
                                       nb, self.stream()), "fcg_nbr_build")
            e_tot = int(c.ptr[-1].item())
            if e_tot <= c.cap_e:
                break
            self.status[_lib.ST_OVERFLOW] = 0
            self._alloc(int(e_tot * 1.5) + 1024)
        c = self.csr
        f_prior = torch.zeros(self.R, self.N, 3, dtype=torch.float32, device=self.device)
        _lib.check(L.fcg_prior_forces(C.byref(self.prior.desc), v(self.pos), self.R, self.N,
                                      v(self.prior_e), v(f_prior), self.stream()),
                   "fcg_prior_forces")
        per_atom = torch.empty(self.R * self.N, dtype=torch.float32, device=self.device)
        ef = L.fcg_ef_workspace_bytes(C.byref(self.model.desc), self.R, self.N, c.cap_e)
        ws_ef = torch.empty(int(ef), dtype=torch.uint8, device=self.device)
        _lib.check(L.fcg_energy_forces_sched(
            C.byref(self.model.desc), v(self.pos), v(self.types), self.R, self.N, v(c.ptr),
            v(c.nbr), v(c.rev), v(c.own), c.cap_e, v(per_atom), v(self.potential), v(self.forces),
            v(ws_ef), ef, self.schedule, self.stream()), "fcg_energy_forces")
        self.model_forces = self.forces.clone()
        self.forces.add_(f_prior)  # out.forces + f_prior, md.py:266
        self.per_atom = per_atom

    def run(self, n_steps: int, graph_steps: int = 0, check: bool = True):
        """Advance n_steps.  With graph_steps > 0, steps run as replays of a
        captured CUDA graph of graph_steps fcg_md_step calls.

        With check=True (the default) the status words are read once at the
        end (one small device->host copy) and a capacity overflow raises
        CapacityError, a blow-up SimulationBlowupError — the step that
        overflowed ran with prior-only forces, so its results are invalid.
        run_simulation repairs both (regrow + replay, blow-up frame); callers
        that batch their own host reads pass check=False and call
        check_status() on the words they copied."""
        if graph_steps <= 0:
            for _ in range(n_steps):
                self._md_step()
        else:
            full, rem = divmod(n_steps, graph_steps)
            if full:
                g = self._graph(graph_steps)
                for _ in range(full):
                    g.replay()
            for _ in range(rem):
                self._md_step()
        if check:
            self.check_status(self.status.cpu().numpy())

    @staticmethod
    def check_status(st) -> None:
        """Raise on the sticky status words of a step batch (include/fcg.h)."""
        if st[_lib.ST_OVERFLOW]:
            raise _lib.CapacityError(
                f"neighbour list overflowed the CSR capacity ({int(st[_lib.ST_EDGES])} edges); "
                "forces of the overflowing steps are invalid — regrow (MDEngine._alloc) and "
                "replay, as run_simulation does")
        if st[_lib.ST_BLOWUP]:
            from .langevin import SimulationBlowupError
            raise SimulationBlowupError(
                f"non-finite or runaway forces at step {int(st[_lib.ST_BLOWUP_STEP])}")

    def _graph(self, k: int):
        g = self._graphs.get(k)
        if g is None:
            torch = self.torch
            # warm the launch path (first-call attribute setup) outside capture
            s = torch.cuda.Stream(self.device)
            g = torch.cuda.CUDAGraph()
            saved = [t.clone() for t in (self.pos, self.vel, self.forces, self.step, self.status)]
            with torch.cuda.graph(g, stream=s):
                for _ in range(k):
                    self._md_step()
            # capture does not execute; restore is a no-op safeguard
            for t, s0 in zip((self.pos, self.vel, self.forces, self.step, self.status), saved):
                t.copy_(s0)
            self._graphs[k] = g
        return g

    def step_host(self, h_state, h_energies=None, h_status=None, n_steps: int = 1):
        """n_steps MD steps from and to host memory as ONE graph launch: the
        state [2, R, N, 3] (positions, velocities) is copied in from pinned
        host memory, the steps run, and the new state, the per-replica
        energies [2, R] (potential, prior) and the status words are copied
        back — the copies are nodes of the same captured CUDA graph
        (fcg_memcpy_async on the capture stream).  Host tensors must be
        pinned and keep their addresses (the graph is cached per address).
        Synchronises; the caller checks the copied status words
        (check_status)."""
        torch, L, v = self.torch, self.lib, _lib.vp
        key = ("host", int(n_steps), h_state.data_ptr(),
               h_energies.data_ptr() if h_energies is not None else 0,
               h_status.data_ptr() if h_status is not None else 0)
        g = self._graphs.get(key)
        if g is None:
            for t in (h_state, h_energies, h_status):
                if t is not None and not t.is_pinned():
                    raise ValueError("step_host needs pinned host tensors")
            if tuple(h_state.shape) != tuple(self.state.shape) or h_state.dtype != self.state.dtype:
                raise ValueError(f"h_state must be {tuple(self.state.shape)} float32")
            s = torch.cuda.Stream(self.device)
            g = torch.cuda.CUDAGraph()
            nb = self.state.numel() * 4
            with torch.cuda.graph(g, stream=s):
                st = self.stream()
                _lib.check(L.fcg_memcpy_async(v(self.state), C.c_void_p(h_state.data_ptr()), nb,
                                              st), "fcg_memcpy_async")
                for _ in range(int(n_steps)):
                    self._md_step()
                _lib.check(L.fcg_memcpy_async(C.c_void_p(h_state.data_ptr()), v(self.state), nb,
                                              st), "fcg_memcpy_async")
                if h_energies is not None:
                    _lib.check(L.fcg_memcpy_async(C.c_void_p(h_energies.data_ptr()),
                                                  v(self.energies), self.energies.numel() * 4,
                                                  st), "fcg_memcpy_async")
                if h_status is not None:
                    _lib.check(L.fcg_memcpy_async(C.c_void_p(h_status.data_ptr()),
                                                  v(self.status), self.status.numel() * 8, st),
                               "fcg_memcpy_async")
            self._graphs[key] = g
        g.replay()
        torch.cuda.current_stream(self.device).synchronize()

    # -- flags -----------------------------------------------------------
    def flags(self):
        st = self.status.cpu().numpy()
        return {"edges": int(st[_lib.ST_EDGES]), "overflow": bool(st[_lib.ST_OVERFLOW]),
                "max_degree": int(st[_lib.ST_MAXDEG]), "blowup": bool(st[_lib.ST_BLOWUP]),
                "blowup_step": int(st[_lib.ST_BLOWUP_STEP]),
                "edge_sum": int(st[_lib.ST_EDGE_SUM]), "builds": int(st[_lib.ST_BUILDS])}

    def clear_flags(self):
        self.status.zero_()
