"""Langevin MD over batched replicas on the GPU — the reference's md.py API
(SimConfig, SimState, integrate, run_simulation, the force-provider
protocol) with every per-step operation in libfcg.so.

Drop-in points (reference md.py):
  * GpuReplicaForces   replaces _ReplicaForces (md.py:231-273): a callable
                       force_fn(positions[R,N,3], step) -> (forces, info)
                       usable by the reference's own integrate();
  * integrate          md.py:188-208: GPU integrator kernels, forces through
                       the host-array force_fn protocol every step;
  * run_simulation     md.py:276-349, device-resident with host I/O only at
                       output strides; same trajectory.xyz / scalars.csv
                       formats, written by a background thread from pinned
                       snapshots (frames formatted in C, fcg_format_xyz);
                       distributed=True shards the replicas over the ranks
                       of torch.distributed (one GPU each).
"""

from __future__ import annotations

import ctypes as C
import math
import queue
import threading
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib
from .engine import KB, MDEngine, md_params
from .schnet import PipelineMode, TrafficReport, accumulated_traffic, io_model_flash_report
from .prior import PriorSpec, DevicePrior  # noqa: F401  (re-export, md.py:90)
from .sharding import ReplicaShards

FORCE_BLOWUP_LIMIT = 1.0e6
SCALARS_SCHEMA = "step,replica,potential,prior,kinetic_T,wall_ms"
NONDETERMINISTIC_COLUMNS = ("wall_ms",)


class SimulationBlowupError(RuntimeError):
    """Non-finite or absurd forces (md.py:37)."""


@dataclass
class SimState:
    positions: np.ndarray
    velocities: np.ndarray
    masses: np.ndarray
    step: int = 0

    @property
    def n_replicas(self) -> int:
        return int(self.positions.shape[0])

    @property
    def n_beads(self) -> int:
        return int(self.positions.shape[1])


@dataclass(frozen=True)
class SimConfig:
    dt_fs: float = 4.0
    temperature: float = 300.0
    friction: float = 1.0
    n_steps: int = 100
    n_replicas: int = 1
    seed: int = 0
    neighbor_stride: int = 1
    output_stride: int = 10
    mode: str = "32bit"
    backend: PipelineMode = field(default_factory=PipelineMode)
    workers: int = 1
    checkpoint_path: str | None = None
    checkpoint_step: int | None = None

    def __post_init__(self):
        if not self.dt_fs > 0:
            raise ValueError("dt must be positive")
        if self.temperature < 0 or self.friction < 0:
            raise ValueError("temperature and friction must be nonnegative")
        if self.mode not in ("32bit", "64bit"):
            raise ValueError(f"unknown mode {self.mode!r}")

    @property
    def dtype(self):
        return np.float64 if self.mode == "64bit" else np.float32

    @property
    def dt_ps(self) -> float:
        return self.dt_fs * 1.0e-3


def _schedule(config: SimConfig) -> int:
    """Aggregation schedule of a fused backend: segment sums, or atomic
    scatter for PipelineMode(fused=True, segred=False) (flash.py:373-443)."""
    return _lib.FCG_SCHED_SEGRED if config.backend.segred else _lib.FCG_SCHED_SCATTER


def _require_fp32(config: SimConfig):
    if config.mode != "32bit":
        raise ValueError("the B200 path integrates in fp32 (mode='32bit'); "
                         "64-bit mode is served by the CPU reference only")


def make_step_rng(seed: int, replica: int, step: int) -> np.random.Generator:
    """Host copy of the counter-based stream the GPU reproduces bitwise
    (md.py:127-131); kept for API parity and debugging."""
    bg = np.random.Philox(key=np.array([seed, replica], dtype=np.uint64),
                          counter=np.array([0, 0, 0, step], dtype=np.uint64))
    return np.random.Generator(bg)


def kinetic_temperature(state: SimState) -> np.ndarray:
    """Per-replica 2 KE / (3 N kB), evaluated as md.py:175-180 does."""
    m = state.masses[None, :, None]
    ke = 0.5 * np.sum(m * state.velocities ** 2, axis=(1, 2))
    return 2.0 * ke / (3 * state.n_beads * KB)


def _check_forces(forces: np.ndarray):
    if not np.all(np.isfinite(forces)) or np.any(np.abs(forces) > FORCE_BLOWUP_LIMIT):
        raise SimulationBlowupError("non-finite or runaway forces")


class GpuReplicaForces:
    """Batched model + prior force provider (replaces md.py:231-273).

    force_fn(positions[R,N,3], step) -> (forces[R,N,3] fp32,
    {"potential": [R], "prior": [R]}): one neighbour rebuild + one fused
    energy/force evaluation for all replicas per call.
    """

    def __init__(self, params, types, prior, config: SimConfig, device="cuda"):
        self.params, self.types, self.prior, self.config = params, np.asarray(types), prior, config
        self.device = device
        self.engine = None
        self.edge_counts = []
        self.traffic = TrafficReport()
        self._cached_step = None

    def _engine_for(self, R: int) -> MDEngine:
        if self.engine is None or self.engine.R != R:
            c = self.config
            self.engine = MDEngine(self.params, self.types, np.full(self.types.size, 1.0),
                                   self.prior, R, c.dt_fs, c.temperature, c.friction, c.seed,
                                   c.neighbor_stride, device=self.device,
                                   schedule=_schedule(c))
        return self.engine

    def __call__(self, positions, step):
        positions = np.asarray(positions)
        R = positions.shape[0]
        fresh = self.engine is None or self.engine.R != R
        eng = self._engine_for(R)
        eng.pos.copy_(eng.torch.as_tensor(positions.astype(np.float32)))
        # md.py:245: rebuild on first use and every neighbor_stride steps
        eng.evaluate(rebuild=fresh or step % max(self.config.neighbor_stride, 1) == 0)
        forces = eng.forces.cpu().numpy()
        info = {"potential": eng.potential.cpu().numpy().astype(np.float64),
                "prior": eng.prior_e.cpu().numpy().astype(np.float64)}
        ptr = eng.csr.ptr.cpu().numpy()
        N = eng.N
        counts = ptr[N::N] - ptr[0:-1:N][:R]
        self.edge_counts.extend(int(x) for x in counts)
        for e in counts:
            self.traffic.merge(accumulated_traffic(self.config.backend, N, int(e), 1,
                                                   self.params))
        return forces.astype(positions.dtype, copy=False), info


def integrate(force_fn, state: SimState, config: SimConfig, observer=None) -> SimState:
    """BAOAB loop with one force evaluation per step (md.py:188-208).

    The integrator runs on the GPU (numpy-exact noise, fp32 BAOA and
    half-kick kernels).  force_fn is called with host arrays each step, as
    the reference protocol defines it, so positions and forces cross the
    host boundary once per step (a GpuReplicaForces evaluates on the GPU);
    run_simulation is the device-resident loop.
    """
    _require_fp32(config)
    from .engine import _torch

    torch = _torch()
    lib = _lib.load()
    R, N = state.n_replicas, state.n_beads
    dev = torch.device("cuda")
    p = md_params(config.dt_fs, config.temperature, config.friction, config.seed)
    mass = torch.as_tensor(np.asarray(state.masses, np.float64).astype(np.float32), device=dev)
    pos = torch.as_tensor(np.asarray(state.positions, np.float32), device=dev).contiguous()
    vel = torch.as_tensor(np.asarray(state.velocities, np.float32), device=dev).contiguous()
    noise = torch.empty_like(pos)
    step_t = torch.tensor([int(state.step)], dtype=torch.int64, device=dev)
    stream = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    v = _lib.vp

    def host_state():
        return SimState(positions=pos.cpu().numpy(), velocities=vel.cpu().numpy(),
                        masses=state.masses, step=int(step_t.item()))

    def eval_forces():
        f, info = force_fn(pos.cpu().numpy(), int(step_t.item()))
        _check_forces(f)
        return torch.as_tensor(np.asarray(f, np.float32), device=dev).contiguous(), f, info

    F, f_host, info = eval_forces()
    if observer is not None:
        observer(host_state(), f_host, info, initial=True)
    for _ in range(config.n_steps):
        _lib.check(lib.fcg_normal_noise(p.seed, 0, v(step_t), R, N, v(noise), stream()),
                   "fcg_normal_noise")
        _lib.check(lib.fcg_langevin_baoa(C.byref(p), v(mass), R, N, v(F), v(noise), v(pos),
                                         v(vel), stream()), "fcg_langevin_baoa")
        step_t += 1
        F, f_host, info = eval_forces()
        _lib.check(lib.fcg_half_kick(C.byref(p), v(mass), R, N, v(F), v(vel), stream()),
                   "fcg_half_kick")
        if observer is not None:
            observer(host_state(), f_host, info, initial=False)
    return host_state()


@dataclass
class RunResult:
    trajectory_path: Path | None
    scalars_path: Path | None
    steps: int
    replicas: int
    wall_seconds: float
    dt_fs: float
    final_state: SimState
    traffic: TrafficReport
    mean_edges: float


def _format_frame(types, positions, step, replica):
    rows = [f"{positions.shape[0]}", f"step={step} replica={replica}"]
    rows += [f"B{int(t)} {x:.9f} {y:.9f} {z:.9f}" for t, (x, y, z) in zip(types, positions)]
    return "\n".join(rows) + "\n"


def _scalar_rows(step, pot, pri, kin, wall_ms, replica0=0) -> str:
    """scalars.csv rows of one output step (md.py:322-326)."""
    return "".join(f"{step},{replica0 + rep},{pot[rep]:.10g},{pri[rep]:.10g},{kin[rep]:.10g},"
                   f"{wall_ms:.3f}\n" for rep in range(len(pot)))


class _FrameWriter:
    """Output pipeline of run_simulation.

    snapshot() enqueues async device->pinned copies of the state on the
    engine's stream and returns at once; a writer thread waits for them,
    computes kinetic T (md.py:175-180), formats the frames in C and appends
    trajectory.xyz / scalars.csv rows in (step, replica) order.  A ring of
    `depth` pinned slots bounds the memory and applies back-pressure.
    """

    def __init__(self, eng, types, masses, traj, scal, depth: int = 3, replica0: int = 0,
                 collect: bool = False):
        torch = eng.torch
        R, N = eng.R, eng.N
        self.eng, self.types, self.masses = eng, np.asarray(types), masses
        self.traj, self.scal = traj, scal
        self.replica0 = replica0
        # collect=True (sharded runs): keep (step, wall_ms, positions,
        # potential, prior, kinetic T) per output instead of writing; rank 0
        # writes every shard's frames after the end-of-run gather
        self.collect = collect
        self.frames = []
        pin = dict(dtype=torch.float32, pin_memory=True)
        self.slots = [dict(pos=torch.empty(R, N, 3, **pin), vel=torch.empty(R, N, 3, **pin),
                           pot=torch.empty(R, **pin), pri=torch.empty(R, **pin),
                           ev=torch.cuda.Event()) for _ in range(depth)]
        self.free = queue.Queue()
        for i in range(depth):
            self.free.put(i)
        self.work = queue.Queue()
        self.error = None
        self.thread = threading.Thread(target=self._run, name="fcg-output", daemon=True)
        self.thread.start()

    def snapshot(self, step: int, wall_ms: float):
        i = self.free.get()
        if self.error is not None:
            raise self.error
        s, e = self.slots[i], self.eng
        s["pos"].copy_(e.pos, non_blocking=True)
        s["vel"].copy_(e.vel, non_blocking=True)
        s["pot"].copy_(e.potential, non_blocking=True)
        s["pri"].copy_(e.prior_e, non_blocking=True)
        s["ev"].record()
        self.work.put((i, step, wall_ms))

    def _run(self):
        while True:
            item = self.work.get()
            if item is None:
                return
            i, step, wall_ms = item
            try:
                if self.error is None:
                    s = self.slots[i]
                    s["ev"].synchronize()
                    pos, vel = s["pos"].numpy(), s["vel"].numpy()
                    st = SimState(positions=pos, velocities=vel, masses=self.masses, step=step)
                    kin = kinetic_temperature(st)
                    pot = s["pot"].numpy().astype(np.float64)
                    pri = s["pri"].numpy().astype(np.float64)
                    if self.collect:
                        self.frames.append((step, wall_ms, pos.copy(),
                                            np.stack([pot, pri, kin], axis=1)))
                    else:
                        self.traj.write(_lib.format_xyz(pos, self.types, step, self.replica0))
                        self.scal.write(_scalar_rows(step, pot, pri, kin, wall_ms,
                                                     self.replica0))
            except BaseException as exc:  # surfaced on the next snapshot/close
                self.error = exc
            finally:
                self.free.put(i)

    def close(self):
        if self.thread.is_alive():
            self.work.put(None)
            self.thread.join()
        if self.error is not None:
            raise self.error


def run_simulation(params, system, config: SimConfig, out_dir, resume_from=None,
                   graph_steps: int = 32, rep_offset: int = 0, distributed: bool = False,
                   group=None) -> RunResult:
    """Device-resident run_simulation (md.py:276-349).

    Frames and scalars are written for the initial state and every
    output_stride steps, ordered by (step, replica), in the reference's
    formats.  Steps between outputs run as CUDA-graph replays; state comes
    back to the host only at outputs, checkpoints and the end.  Capacity
    overflow is repaired by regrowing the CSR buffers and replaying the
    chunk from its saved start state (results are unchanged: the noise is
    counter-based).  A blow-up dumps the frame of the offending step to
    blowup.xyz and raises SimulationBlowupError.

    distributed=True: the n_replicas replicas are sharded over
    the ranks of torch.distributed (`group`, default the world; each rank
    drives its current CUDA device).  Rank g integrates the contiguous block
    sharding.replica_shard gives it, with its first global replica index
    keying the noise (md.py:127-131), so no per-step exchange exists.  The
    ranks meet once per output chunk for one integer (the earliest blow-up
    step) and once at the end, where one gather of the recorded frames,
    per-replica scalars and final states lets rank 0 write the same
    trajectory.xyz / scalars.csv an unsharded run writes (wall_ms is rank
    0's clock).  Every rank returns the full RunResult.
    """
    from . import checkpoint as params_io

    _require_fp32(config)
    if not config.backend.fused:
        if distributed:
            raise ValueError("distributed runs use the fused backend")
        return _run_simulation_materialized(params, system, config, out_dir, resume_from)
    out_dir = Path(out_dir)
    shard = ReplicaShards(config.n_replicas, group) if distributed else None
    lead = shard is None or shard.rank == 0
    if lead:
        out_dir.mkdir(parents=True, exist_ok=True)
    masses = np.asarray(system.masses, np.float64)
    if resume_from is not None:
        chk = params_io.load_checkpoint(resume_from)
        pos0 = chk["positions"].astype(np.float32)
        vel0 = chk["velocities"].astype(np.float32)
        masses = chk["masses"].astype(np.float64)
        step0 = int(chk["step"])
    else:
        r0 = system.initial_positions()
        pos0 = np.repeat(r0[None, :, :], config.n_replicas, axis=0).astype(np.float32)
        vel0 = np.zeros_like(pos0)
        step0 = 0
    R_total, N = pos0.shape[0], pos0.shape[1]
    first = 0
    if shard is not None:
        if R_total != config.n_replicas:
            raise ValueError("checkpoint replica count differs from config.n_replicas")
        first, cnt = shard.first, shard.count
        pos0, vel0 = pos0[first:first + cnt], vel0[first:first + cnt]
    R = pos0.shape[0]
    eng = MDEngine(params, system.types, masses, system.prior, R, config.dt_fs,
                   config.temperature, config.friction, config.seed, config.neighbor_stride,
                   rep_offset=rep_offset + first, schedule=_schedule(config))
    eng.load_state(pos0, vel0, step0)

    traj_path, scal_path = out_dir / "trajectory.xyz", out_dir / "scalars.csv"
    traj = scal = None
    if shard is None:
        traj = open(traj_path, "wb")
        scal = open(scal_path, "w")
        scal.write("# flashcg-scalars v1\n" + SCALARS_SCHEMA + "\n")
    writer = _FrameWriter(eng, system.types, masses, traj, scal, collect=shard is not None)
    t_start = time.perf_counter()
    last = [t_start]
    edge_total = [0, 0]  # (sum of per-replica edge counts, evaluations*replicas)

    def emit(step_done: int, steps_since: int):
        now = time.perf_counter()
        wall_ms = (now - last[0]) * 1e3 / max(steps_since, 1)
        last[0] = now
        writer.snapshot(step_done, wall_ms)

    def close_files():
        for f in (traj, scal):
            if f is not None:
                f.close()

    def blowup(step_at):
        writer.close()  # frames before the blow-up are complete
        pos = eng.pos.cpu().numpy()
        if shard is not None:
            pos = shard.gather(pos)
        dump = out_dir / "blowup.xyz"
        if lead:
            with open(dump, "wb") as f:
                f.write(_lib.format_xyz(pos, system.types, step_at))
        close_files()
        raise SimulationBlowupError(f"simulation blew up at step {step_at}; "
                                    f"diagnostic frame in {dump}")

    def checkpoint(at):
        p, v_ = eng.pos.cpu().numpy(), eng.vel.cpu().numpy()
        if shard is not None:
            p, v_ = shard.gather(p), shard.gather(v_)
        if lead:
            params_io.save_checkpoint(config.checkpoint_path, p, v_, masses, at, config.seed)

    NO_BLOWUP = 2 ** 62
    try:
        eng.evaluate()
        f0 = eng.forces.cpu().numpy()
        edge_total[0] += int(eng.csr.ptr[-1].item())
        edge_total[1] += R
        bad0 = not np.all(np.isfinite(f0)) or np.any(np.abs(f0) > FORCE_BLOWUP_LIMIT)
        if shard is not None:
            bad0 = shard.min_int(step0 if bad0 else NO_BLOWUP) != NO_BLOWUP
        if bad0:
            blowup(step0)
        if config.checkpoint_step is not None and step0 == config.checkpoint_step \
                and config.checkpoint_path:
            checkpoint(step0)
        emit(step0, 1)
        stride = max(config.output_stride, 1)
        cur, end = step0, step0 + config.n_steps
        while cur < end:
            nxt = min(end, (cur // stride + 1) * stride)
            if config.checkpoint_step is not None and cur < config.checkpoint_step < nxt:
                nxt = config.checkpoint_step
            n = nxt - cur
            saved = [t.clone() for t in (eng.pos, eng.vel, eng.forces, eng.step)]
            csr0 = eng.save_csr() if config.neighbor_stride > 1 else None
            eng.clear_flags()
            eng.run(n, graph_steps=min(graph_steps, n) if n >= 4 else 0, check=False)
            fl = eng.flags()
            if fl["overflow"]:   # local repair: regrow and replay the chunk
                for t, s0 in zip((eng.pos, eng.vel, eng.forces, eng.step), saved):
                    t.copy_(s0)
                eng._alloc(max(2 * eng.cap_e, int(1.5 * fl["edges"]) + 1024), keep=csr0)
                continue
            # the earliest blow-up step over all shards stops every shard there
            b_step = fl["blowup_step"] if fl["blowup"] else NO_BLOWUP
            if shard is not None:
                b_step = shard.min_int(b_step)
            if b_step != NO_BLOWUP:
                for t, s0 in zip((eng.pos, eng.vel, eng.forces, eng.step), saved):
                    t.copy_(s0)
                if csr0 is not None:
                    eng._alloc(eng.cap_e, keep=csr0)
                eng.clear_flags()
                # replay one step at a time up to the blow-up step
                while int(eng.step.item()) < b_step:
                    eng.run(1, check=False)
                    if shard is None and eng.flags()["blowup"]:
                        break
                blowup(int(eng.step.item()))
            edge_total[0] += fl["edge_sum"]
            edge_total[1] += fl["builds"] * R
            cur = nxt
            if config.checkpoint_step is not None and cur == config.checkpoint_step \
                    and config.checkpoint_path:
                checkpoint(cur)
            if cur % stride == 0:
                emit(cur, n)
        eng.torch.cuda.synchronize()
        writer.close()
    finally:
        if writer.thread.is_alive():
            writer.work.put(None)
            writer.thread.join()
        close_files()

    pos, vel, step = eng.read_state()
    if shard is not None:
        # the end-of-run exchange: final states, recorded frames and scalars
        pos, vel = shard.gather(pos), shard.gather(vel)
        frames = writer.frames
        fpos = shard.gather(np.stack([f[2] for f in frames], axis=1))    # [R, F, N, 3]
        fsc = shard.gather(np.stack([f[3] for f in frames], axis=1))     # [R, F, 3]
        edge_total = [int(x) for x in shard.sum_int(edge_total)]
        if lead:
            with open(traj_path, "wb") as traj_f, open(scal_path, "w") as scal_f:
                scal_f.write("# flashcg-scalars v1\n" + SCALARS_SCHEMA + "\n")
                for k, (st, wall_ms, _, _) in enumerate(frames):
                    traj_f.write(_lib.format_xyz(fpos[:, k], system.types, st))
                    scal_f.write(_scalar_rows(st, fsc[:, k, 0], fsc[:, k, 1], fsc[:, k, 2],
                                              wall_ms))
        shard.barrier()
        R = R_total
    wall = time.perf_counter() - t_start
    mean_edges = edge_total[0] / edge_total[1] if edge_total[1] else 0.0
    evaluations = R * (config.n_steps + 1)   # integrate(): one evaluation per step + initial
    traffic = accumulated_traffic(config.backend, N, round(mean_edges * evaluations),
                                  evaluations, params)
    return RunResult(trajectory_path=traj_path, scalars_path=scal_path, steps=config.n_steps,
                     replicas=R, wall_seconds=wall, dt_fs=config.dt_fs,
                     final_state=SimState(positions=pos, velocities=vel, masses=masses, step=step),
                     traffic=traffic, mean_edges=mean_edges)


def _run_simulation_materialized(params, system, config: SimConfig, out_dir, resume_from=None):
    """run_simulation under a fused=False backend (the reference's ablation
    cells, bench.py:121-192): the reference observer loop over integrate()
    with the GPU integrator and GPU materialising forces (ablation.py)."""
    from . import checkpoint as params_io
    from .ablation import MaterializedReplicaForces

    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    masses = np.asarray(system.masses, np.float64)
    if resume_from is not None:
        chk = params_io.load_checkpoint(resume_from)
        pos0, vel0 = chk["positions"].astype(np.float32), chk["velocities"].astype(np.float32)
        masses, step0 = chk["masses"].astype(np.float64), int(chk["step"])
    else:
        r0 = system.initial_positions()
        pos0 = np.repeat(r0[None, :, :], config.n_replicas, axis=0).astype(np.float32)
        vel0, step0 = np.zeros_like(pos0), 0
    state = SimState(positions=pos0, velocities=vel0, masses=masses, step=step0)
    provider = MaterializedReplicaForces(params, system.types, system.prior, config,
                                         segred=config.backend.segred)
    traj_path, scal_path = out_dir / "trajectory.xyz", out_dir / "scalars.csv"
    traj = open(traj_path, "wb")
    scal = open(scal_path, "w")
    scal.write("# flashcg-scalars v1\n" + SCALARS_SCHEMA + "\n")
    t_start = time.perf_counter()
    last = [t_start]

    def observer(st, forces, info, initial):  # md.py:312-326
        now = time.perf_counter()
        wall_ms = (now - last[0]) * 1e3
        last[0] = now
        if config.checkpoint_step is not None and st.step == config.checkpoint_step \
                and config.checkpoint_path:
            params_io.save_checkpoint(config.checkpoint_path, st.positions, st.velocities,
                                      st.masses, st.step, config.seed)
        if not (initial or st.step % max(config.output_stride, 1) == 0):
            return
        kin = kinetic_temperature(st)
        traj.write(_lib.format_xyz(st.positions, system.types, st.step))
        scal.write("".join(f"{st.step},{rep},{info['potential'][rep]:.10g},"
                           f"{info['prior'][rep]:.10g},{kin[rep]:.10g},{wall_ms:.3f}\n"
                           for rep in range(st.n_replicas)))

    try:
        state = integrate(provider, state, config, observer=observer)
    except SimulationBlowupError:  # md.py:330-339 (dumps the state it holds)
        dump = out_dir / "blowup.xyz"
        with open(dump, "wb") as f:
            f.write(_lib.format_xyz(state.positions, system.types, state.step))
        raise SimulationBlowupError(
            f"simulation blew up at step {state.step}; diagnostic frame in {dump}")
    finally:
        traj.close()
        scal.close()
    wall = time.perf_counter() - t_start
    counts = provider.edge_counts
    return RunResult(trajectory_path=traj_path, scalars_path=scal_path, steps=config.n_steps,
                     replicas=state.n_replicas, wall_seconds=wall, dt_fs=config.dt_fs,
                     final_state=state, traffic=provider.traffic,
                     mean_edges=float(np.mean(counts)) if counts else 0.0)


def throughput_report(result: RunResult) -> dict:
    """timestep*mol/s and ns/day (md.py:352-364)."""
    if result.wall_seconds <= 0:
        raise ValueError("cannot report throughput for a run with zero elapsed time")
    rate = result.steps * result.replicas / result.wall_seconds
    return {"steps": result.steps, "replicas": result.replicas,
            "wall_seconds": result.wall_seconds, "timestep_mol_per_s": rate,
            "ns_per_day": rate * result.dt_fs * 86400.0 / 1.0e6}
