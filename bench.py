#!/usr/bin/env python
"""Benchmark: aggregate ns/day of the IO-aware SchNet MD step (BASELINE.json).

Workload (BASELINE configs[1], weak-scaled per configs[3]): the 1ENH
stand-in generate_system("coil", 269, 0) (SURVEY §7 hard part 6), random
init_params(ModelConfig(), 0) weights (D=128, D_r=64, T=3, r_cut=1.5 nm),
64 replicas per GPU, fp32, dt=4 fs, 300 K, friction 1/ps, neighbour list
rebuilt every step.  A "step" is one full MD step of all replicas (noise,
BAOA, neighbour/CSR rebuild, prior, energy + force backward, half-kick).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config fp32|w16]
    python bench.py --impl reference ...   # the reference's CPU implementation

--gpus N > 1 without torchrun around it relaunches itself under
torch.distributed.run with N ranks (one per GPU); under torchrun,
WORLD_SIZE must equal --gpus.

Timing: W untimed warm-up steps, then K steps, each a replay of a captured
one-step CUDA graph bracketed by CUDA events on the replay stream, with a
256 MiB L2 flush (outside the events) before every step; barrier +
synchronize around the timed region; max over ranks.  `e2e` repeats the
step through the engine's public host-buffer call MDEngine.step_host (H2D
of positions+velocities from pinned memory, fcg_md_step, D2H of the new
state, per-replica energies and status words — one graph launch whose
copies are graph nodes), timed by the host clock around each call's
synchronisation and status check.  Multi-GPU: one process per GPU, replicas
sharded with no per-step collective; after the timed region one NCCL
all_gather of the final positions, velocities and per-replica potential,
prior and kinetic T.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

DT_FS = 4.0
METRIC = "aggregate ns/day (64 replicas, 269-bead 1ENH) per GPU and at 1/2/4/8 B200; peak mem"
UNIT = "ns/day"


def ns_per_day(replica_steps: float, seconds: float) -> float:
    return replica_steps / seconds * DT_FS * 86400.0 / 1.0e6


def workload(config: str, system: str = "coil", beads: int = 269, cutoff: float = 1.5):
    from paper_2602_13140_b200.inputs import generate_system
    from paper_2602_13140_b200.modelparams import ModelConfig, init_params

    # BASELINE configs[4] stress variant: unbonded globule
    sysm = generate_system(system, beads, 0, bonded=(system != "globule"))
    params = init_params(ModelConfig(cutoff=cutoff), 0)
    if config == "w16":
        from paper_2602_13140_b200.w16 import quantize_model
        params = quantize_model(params, seed=0)
    return sysm, params


def flops_per_edge_block():
    """Algorithmic filter-MLP FLOPs per edge per block and pass:
    2*(D_r*F_h + F_h*D) = 49,152 for the forward, same for the backward."""
    return 2 * (64 * 128 + 128 * 128)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", gpu_id, "-lms", "100"], stdout=self.tmp, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = [r.split(", ") for r in Path(self.tmp.name).read_text().splitlines() if r.strip()]
        os.unlink(self.tmp.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows if len(r) >= 9
                          for k in range(4) if r[5 + k].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def config_tag(args) -> str:
    """Key of this workload in profiles/ncu_summary.json."""
    return f"{args.system}{args.beads}_rc{args.cutoff:g}_{args.config}_R{args.replicas}"


def load_flashcg():
    """The unmodified reference package installed into baseline/_ref
    (pip --target), or None when it is not there."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "flashcg" / "md.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import importlib
    mods = {m: importlib.import_module(f"flashcg.{m}") for m in ("md", "model", "quantize",
                                                                 "systems")}
    return mods


def reference_run(args, replicas: int, budget_s: float, max_steps: int, workers: int,
                  blas_threads: int):
    """Time the reference's own run_simulation (md.py:276-349) through its
    public API on this host: `replicas` replicas of the bench workload,
    `workers` replica threads x `blas_threads` BLAS threads, one warm-up
    step, then as many steps (<= max_steps) as fit in budget_s.  Returns
    (ns/day from the reference's throughput_report, steps, seconds, kind)."""
    from threadpoolctl import threadpool_limits

    fc = load_flashcg()
    with tempfile.TemporaryDirectory() as td, threadpool_limits(limits=blas_threads):
        if fc is not None:
            md, model = fc["md"], fc["model"]
            sysm = fc["systems"].generate_system(args.system, args.beads, 0,
                                                 bonded=(args.system != "globule"))
            params = model.init_params(model.ModelConfig(cutoff=args.cutoff), 0)
            if args.config == "w16":
                params = fc["quantize"].quantize_model(params, seed=0)

            def run(n):
                cfg = md.SimConfig(dt_fs=DT_FS, temperature=300.0, friction=1.0, n_steps=n,
                                   n_replicas=replicas, seed=0, neighbor_stride=1,
                                   output_stride=max(n, 1), workers=workers)
                res = md.run_simulation(params, sysm, cfg, td)
                return md.throughput_report(res)["ns_per_day"], res.wall_seconds
            kind = "reference"
        else:  # the oracle port of the same numpy algorithm (oracle/flashcg_oracle.py)
            sysm, params = workload(args.config, args.system, args.beads, args.cutoff)

            def run(n):
                ref = CpuReference(sysm, params, replicas, workers)
                t0 = time.perf_counter()
                for _ in range(n):
                    ref.step()
                dt = time.perf_counter() - t0
                return ns_per_day(replicas * n, dt), dt
            kind = "port"
        _, warm_s = run(1)                       # warm-up (includes the initial evaluation)
        per_step = warm_s / 2.0
        steps = int(max(1, min(max_steps, budget_s // max(per_step, 1e-9))))
        value, secs = run(steps)
    return value, steps, secs, kind


class CpuReference:
    """Oracle port of the reference step (numpy + BLAS, same ops as flashcg),
    used only when baseline/_ref holds no reference install."""

    def __init__(self, sysm, params, replicas: int, workers: int):
        from oracle import flashcg_oracle as O

        self.O, self.sysm, self.params, self.R, self.workers = O, sysm, params, replicas, workers
        self.pos = np.repeat(sysm.positions[None], replicas, axis=0).astype(np.float32)
        self.vel = np.zeros_like(self.pos)
        self.step_idx = 0
        self.F, *_ = O.replica_forces(params, sysm.types, sysm.prior, self.pos, workers)

    def step(self):
        O, s = self.O, self.sysm
        xi = np.stack([O.noise(0, r, self.step_idx, s.n_beads) for r in range(self.R)])
        self.pos, self.vel = O.baoa(self.pos, self.vel, self.F, s.masses, xi, DT_FS, 300.0, 1.0)
        self.F, *_ = O.replica_forces(self.params, s.types, s.prior, self.pos, self.workers)
        self.vel = O.half_kick(self.vel, self.F, s.masses, DT_FS)
        self.step_idx += 1


def cpu_baseline(args, budget_s: float = 20.0):
    """cpu_baseline of our line: the reference CPU path on this host's cores,
    a bounded sample of the same 64-replica workload (SURVEY §8(d) mode 2)."""
    cores = os.cpu_count() or 1
    value, steps, secs, kind = reference_run(args, args.replicas, budget_s, 5, cores, 1)
    src = ("flashcg.md.run_simulation from baseline/_ref (unmodified reference)"
           if kind == "reference" else "oracle port of the reference algorithm")
    return {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{args.replicas} replicas x {steps} full MD steps of {args.system}-"
                      f"{args.beads} ({secs:.1f} s incl. the initial evaluation; {src}, numpy "
                      f"{np.__version__}, {cores} replica threads x 1 BLAS thread)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    R = args.replicas
    # SURVEY §8(d) CPU mode 2: all replicas of the workload, one thread per
    # core, 1 BLAS thread each; steps bounded by --ref-budget-s
    value, steps, secs, kind = reference_run(args, R, args.ref_budget_s, args.steps, cores, 1)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": steps, "steps_requested": args.steps,
            "warmup": 1, "ms_per_step": secs / steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.system}-{args.beads} (1ENH stand-in) x {R} replicas, "
                                   f"r_cut={args.cutoff} nm, dt=4 fs, nbr rebuild every step",
                       "replicas": R, "same_config": True,
                       "weights": "init_params(ModelConfig(), 0)" + (
                           " + quantize_model" if args.config == "w16" else ""),
                       "path": ("flashcg.md.run_simulation (baseline/_ref, unmodified), "
                                "throughput_report" if kind == "reference"
                                else "oracle port (baseline/_ref missing)")},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": f"{R} replicas x {steps} steps ({secs:.1f} s, "
                                       f"{cores} replica threads x 1 BLAS thread)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if (args.system, args.beads, args.config) == ("coil", 269, "fp32") and not args.no_c1:
        # BASELINE configs[0] / SURVEY §8(d) mode 1: one replica, all cores on BLAS
        c1, c1_steps, c1_s, c1_kind = reference_run(args, 1, 30.0, 100, 1, cores)
        line["c1"] = {"value": c1, "unit": UNIT, "replicas": 1, "steps": c1_steps,
                      "seconds": c1_s, "kind": c1_kind, "blas_threads": cores,
                      "workload": "BASELINE configs[0]: 1 replica of coil-269, up to 100 "
                                  "Langevin steps fp32"}
    print(json.dumps(line), flush=True)


def graph_kernel_nodes(g):
    """Kernel nodes of the captured one-step CUDA graph (every launch of a
    timed step); None if the graph cannot be inspected."""
    try:
        from cuda.bindings import runtime as rt
        raw = g.raw_cuda_graph()
        err, _, n = rt.cudaGraphGetNodes(raw, numNodes=0)
        err, nodes, n = rt.cudaGraphGetNodes(raw, numNodes=n)
        kernel = rt.cudaGraphNodeType.cudaGraphNodeTypeKernel
        return sum(1 for nd in nodes if rt.cudaGraphNodeGetType(nd)[1] == kernel)
    except Exception:
        return None


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch(args) -> int:
    """`python bench.py --gpus N` without a launcher: run N ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def step_roofline(E_tot: int, R: int, N: int, params, ms_step: float, pk: dict, w16: bool):
    """SURVEY §8(d) whole-step roofline: algorithmic bytes (io_model_flash,
    summed over replicas, + integrator/neighbour bytes) against HBM, and
    algorithmic FLOPs against the FP32 FFMA and bf16 tensor peaks; names the
    bound whose time is larger for the pipes the kernels use."""
    from paper_2602_13140_b200.schnet import PipelineMode, accumulated_traffic

    cfg = params.config
    D, Dr, Fh, Rh, T = (cfg.hidden_dim, cfg.rbf_dim, cfg.filter_hidden_dim,
                        cfg.readout_hidden_dim, cfg.num_blocks)
    width = 2 if w16 else 4
    bytes_alg = accumulated_traffic(PipelineMode(), N, E_tot, R, params, width).total_bytes
    bytes_alg += R * N * 3 * 4 * 6            # integrator: pos/vel read+write, forces, noise
    flop_alg = (2 * T * E_tot * 2 * (Dr * Fh + Fh * D) + R * 12 * T * N * D * D
                + R * 4 * N * (D * Rh + Rh))
    t = ms_step / 1e3
    ffma = 148 * 128 * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6
    hbm = pk["hbm_gbs"] * 1e9
    tensor = pk["bf16_tflops"] * 1e12
    # the fp32 path issues 3 fp16 products per MAC (hi*hi + hi*lo + lo*hi)
    issued = flop_alg * (1 if w16 else 3)
    t_hbm, t_tensor = bytes_alg / hbm, issued / tensor
    return {"bytes_alg": int(bytes_alg), "achieved_gbs": bytes_alg / t / 1e9,
            "hbm_frac": bytes_alg / t / hbm,
            "flop_alg": int(flop_alg), "achieved_tflops": flop_alg / t / 1e12,
            "ffma_frac": flop_alg / t / ffma, "tensor_frac": flop_alg / t / tensor,
            "tensor_issued_frac": issued / t / tensor,
            "bound": "hbm" if t_hbm >= t_tensor else "tensor",
            "bound_ms": max(t_hbm, t_tensor) * 1e3, "frac_of_bound": max(t_hbm, t_tensor) / t,
            "note": ("bytes: io_model_flash at width %d B summed over replicas + 72 B/bead "
                     "integrator; FLOPs: SURVEY §8(d) FLOP_alg; fp32 path issues 3 fp16 tensor "
                     "products per MAC (hi/lo split)" % width)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=("fp32", "w16"), default="fp32")
    ap.add_argument("--replicas", type=int, default=64, help="replicas per GPU")
    ap.add_argument("--system", choices=("coil", "globule"), default="coil")
    ap.add_argument("--beads", type=int, default=269)
    ap.add_argument("--cutoff", type=float, default=1.5)
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--profile-steps", type=int, default=3)
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gpu-baseline", action="store_true",
                    help="skip the same-GPU materialising (CGSchNet-style) comparison")
    ap.add_argument("--no-c1", action="store_true", help="reference arm: skip the C1 run")
    ap.add_argument("--ref-budget-s", type=float, default=120.0,
                    help="reference arm: seconds of timed CPU steps (bounded sample)")
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl")
    ap.add_argument("--share-gpu", action="store_true",
                    help="all ranks on cuda:0 (tests of the launcher on a 1-GPU box; gloo)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2602_13140_b200 import _lib
    from paper_2602_13140_b200.engine import KB, MDEngine

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(0 if args.share_gpu else local)
    dev = torch.device("cuda", torch.cuda.current_device())
    if world > 1:
        dist.init_process_group(args.dist_backend,
                                **({"device_id": dev} if args.dist_backend == "nccl" else {}))

    sysm, params = workload(args.config, args.system, args.beads, args.cutoff)
    R, N = args.replicas, sysm.n_beads
    eng = MDEngine(params, sysm.types, sysm.masses, sysm.prior, R, dt_fs=DT_FS, seed=0,
                   rep_offset=rank * R, device=dev)
    pos0 = np.repeat(sysm.positions[None], R, axis=0).astype(np.float32)
    eng.load_state(pos0, np.zeros_like(pos0), 0)
    eng.evaluate()
    torch.cuda.reset_peak_memory_stats(dev)
    g = eng._graph(1)
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64,
                         device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            g.replay()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        torch.cuda.synchronize(dev)
        barrier()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        gpu_index = dev.index
        sampler = ClockSampler(vis.split(",")[gpu_index] if vis else str(gpu_index))
        for s0, s1 in evs:
            if not args.no_flush:
                flush.zero_()
            s0.record(stream)
            g.replay()
            s1.record(stream)
        torch.cuda.synchronize(dev)
        clocks = sampler.stop()
        barrier()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    peak_mem = torch.cuda.max_memory_allocated(dev)
    ms_max = max_over_ranks(ms)
    value = ns_per_day(R * world * args.steps, ms_max / 1e3)
    st_np = eng.status.cpu().numpy()
    MDEngine.check_status(st_np)   # an overflow or blow-up would void the timing

    # ---- end-to-end through the host-buffer API --------------------------
    hstate = torch.empty((2, R, N, 3), dtype=torch.float32).pin_memory()  # positions, velocities
    hen = torch.empty((2, R), dtype=torch.float32).pin_memory()            # potential, prior
    hst = torch.empty(_lib.FCG_STATUS_WORDS, dtype=torch.int64).pin_memory()
    hstate.copy_(eng.state)
    with torch.cuda.stream(stream):
        # the public host-buffer stepping call: state in from pinned host
        # memory, one MD step, state + energies + status back, as one graph
        # launch (MDEngine.step_host); the first call captures it
        eng.step_host(hstate, hen, hst)
        MDEngine.check_status(hst.numpy())
        torch.cuda.synchronize(dev)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            eng.step_host(hstate, hen, hst)
            MDEngine.check_status(hst.numpy())
        e2e_s = time.perf_counter() - t0
    e2e_value = ns_per_day(R * world * args.e2e_steps, max_over_ranks(e2e_s))
    h2d = 2 * R * N * 3 * 4
    d2h = 2 * R * N * 3 * 4 + 2 * R * 4 + _lib.FCG_STATUS_WORDS * 8

    # ---- per-kernel device times (built-in profiler, eager steps) ---------
    lib = _lib.load()
    lib.fcg_profile_enable(1)
    with torch.cuda.stream(stream):
        for _ in range(args.profile_steps):
            eng._md_step()
    prof = _lib.profile_read()
    lib.fcg_profile_enable(0)
    flags = eng.flags()
    E_tot = flags["edges"]
    per_step_launch = graph_kernel_nodes(g)
    if per_step_launch is None:  # estimate from the profiler's launch brackets
        per_step_launch = sum(c for _, c in prof.values()) / args.profile_steps
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dom_name, (dom_ms, dom_n) = dom
    avg_ms = dom_ms / dom_n
    pk, pk_kind = peaks()
    if dom_name in ("edge_fwd", "edge_bwd"):
        alg = E_tot * flops_per_edge_block()
        achieved = alg / (avg_ms / 1e3) / 1e12
        roof = {"kernel": dom_name, "bound": "tensor", "achieved": achieved,
                "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": achieved / pk["bf16_tflops"],
                "peak_kind": f"{pk_kind} bf16 dense burst (MEASURED_PEAKS.json bf16_tflops; the "
                             "kernel's launch time is measured on its own)",
                "alg_per_launch": f"{alg:.4g} FLOP = E_total {E_tot} x 49,152 "
                                  "(filter-MLP GEMMs of one pass, SURVEY §8(d))",
                "avg_launch_ms": avg_ms,
                "fp32_ffma_peak_tflops": 148 * 128 * 2 * pk.get("sm_max_mhz", 1965.0) / 1e6,
                "frac_of_fp32_ffma_peak": achieved / (148 * 128 * 2 * pk.get("sm_max_mhz", 1965.0)
                                                      / 1e6)}
    else:
        roof = {"kernel": dom_name, "bound": "hbm", "achieved": None, "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": None, "avg_launch_ms": avg_ms}
    ncu = ROOT / "profiles" / "ncu_summary.json"
    roof["traffic"] = None
    tag = config_tag(args)
    if ncu.exists():
        try:
            ent = json.loads(ncu.read_text()).get(tag, {}).get(dom_name)
            if ent:
                roof["traffic"] = ent["dram_bytes"]
                roof["traffic_source"] = f"profiles/ncu_summary.json[{tag}] (ncu {ent['tag']})"
        except Exception:
            pass
    share = {k: round(v[0] / sum(x[0] for x in prof.values()), 4) for k, v in prof.items()}
    step_roof = step_roofline(E_tot, R, N, params, ms_max / args.steps, pk, args.config == "w16")

    # ---- end-of-run gather of final states and per-replica observables ---
    gdev = dev if args.dist_backend == "nccl" else torch.device("cpu")
    m = eng.mass.double()[None, :, None]
    kin = (2.0 * (0.5 * (m * eng.vel.double() ** 2).sum(dim=(1, 2))) / (3 * N * KB))
    obs = torch.stack([eng.potential.double(), eng.prior_e.double(), kin], dim=1).to(gdev)
    st = eng.state.transpose(0, 1).contiguous().to(gdev)     # [R, 2, N, 3]
    torch.cuda.synchronize(dev)
    barrier()
    t0 = time.perf_counter()
    if world > 1:
        from paper_2602_13140_b200.sharding import gather_replicas
        obs = gather_replicas(obs, R * world)
        st = gather_replicas(st, R * world)
    torch.cuda.synchronize(dev)
    gather_ms = (time.perf_counter() - t0) * 1e3
    gather = {"replicas": int(obs.shape[0]), "what": "final positions+velocities [R,2,N,3] f32 "
              "and per-replica potential, prior, kinetic_T [R,3] f64 (SURVEY §8(e))",
              "bytes": int(st.numel() * 4 + obs.numel() * 8), "ms": gather_ms,
              "backend": args.dist_backend if world > 1 else None}

    if rank == 0:
        sysline = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                   "steps": args.steps, "warmup": max(args.warmup, 3),
                   "ms_per_step": ms_max / args.steps,
                   "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                   "dtype": "f32" if args.config == "fp32" else "f16-weights/f32-accum",
                   "data": "synthetic (generate_system coil-269 seed 0; random-init weights)",
                   "config": {"workload": (f"1ENH stand-in coil-269, {R} replicas/GPU, T=3 D=128 "
                                           f"D_r=64 r_cut={args.cutoff} nm, dt=4 fs, nbr rebuild "
                                           "every step") if (args.system, args.beads) == ("coil", 269)
                              else (f"{args.system}-{args.beads} (BASELINE configs[4] sweep), "
                                    f"{R} replicas/GPU, r_cut={args.cutoff} nm, dt=4 fs"),
                              "tag": tag, "replicas_per_gpu": R, "total_replicas": R * world,
                              "weights": args.config, "parallelism": f"replica-shard x{world}",
                              "l2": "flushed (256 MiB write) before every timed step"
                                    if not args.no_flush else "not flushed",
                              "mean_edges_per_replica": E_tot / R,
                              **({"shared_gpu": True} if args.share_gpu else {})},
                   "gpu_launches": int(round(per_step_launch * args.steps)),
                   "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                           "d2h_bytes_per_step": d2h, "steps": args.e2e_steps},
                   "roofline": roof, "step_roofline": step_roof, "clocks": clocks,
                   "kernel_share": share,
                   "peak_mem_bytes": int(peak_mem),
                   "flags": {k: flags[k] for k in ("overflow", "blowup", "max_degree")},
                   "end_of_run_gather": gather,
                   "energy_mean": float(obs[:, 0].mean().item())}
        if world == 1 and not args.no_gpu_baseline:
            from paper_2602_13140_b200.ablation import compare_on_engine
            sysline["gpu_materialized_baseline"] = compare_on_engine(eng, params)
        if world == 1 and not args.no_cpu_baseline:
            sysline["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(sysline), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
