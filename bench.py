#!/usr/bin/env python
"""Benchmark: aggregate ns/day of the IO-aware SchNet MD step (BASELINE.json).

Workload (BASELINE configs[1], weak-scaled per configs[3]): the 1ENH
stand-in generate_system("coil", 269, 0) (SURVEY §7 hard part 6), random
init_params(ModelConfig(), 0) weights (D=128, D_r=64, T=3, r_cut=1.5 nm),
64 replicas per GPU, fp32, dt=4 fs, 300 K, friction 1/ps, neighbour list
rebuilt every step.  A "step" is one full MD step of all replicas (noise,
BAOA, neighbour/CSR rebuild, prior, energy + force backward, half-kick).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config fp32|w16]
    python bench.py --impl reference ...   # the reference's CPU algorithm

Timing: W untimed warm-up steps, then K steps, each a replay of a captured
one-step CUDA graph bracketed by CUDA events on the replay stream, with a
256 MiB L2 flush (outside the events) before every step; barrier +
synchronize around the timed region; max over ranks.  `e2e` repeats the
step through the engine's public API with host buffers (H2D of
positions+velocities from pinned memory, MDEngine.run(1) = one graph replay
of fcg_md_step, D2H of the new state and per-replica energies) timed by the
host clock.  Multi-GPU: one process per GPU
(torchrun), replicas sharded with no per-step collective; an NCCL
all_gather of per-replica energies happens after the timed region.
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


class CpuReference:
    """The reference algorithm on this host's cores (oracle port: numpy +
    BLAS, same ops as flashcg): replicas spread over a thread pool with one
    BLAS thread each — the reference's CPU-64 mode."""

    def __init__(self, sysm, params, replicas: int):
        from oracle import flashcg_oracle as O

        self.O, self.sysm, self.params, self.R = O, sysm, params, replicas
        self.cores = os.cpu_count() or 1
        self.pos = np.repeat(sysm.positions[None], replicas, axis=0).astype(np.float32)
        self.vel = np.zeros_like(self.pos)
        self.step_idx = 0
        self.F, *_ = O.replica_forces(params, sysm.types, sysm.prior, self.pos, self.cores)

    def step(self):
        O, s = self.O, self.sysm
        xi = np.stack([O.noise(0, r, self.step_idx, s.n_beads) for r in range(self.R)])
        self.pos, self.vel = O.baoa(self.pos, self.vel, self.F, s.masses, xi, DT_FS, 300.0, 1.0)
        self.F, *_ = O.replica_forces(self.params, s.types, s.prior, self.pos, self.cores)
        self.vel = O.half_kick(self.vel, self.F, s.masses, DT_FS)
        self.step_idx += 1


def cpu_baseline(sysm, params, replicas: int, max_seconds: float = 20.0, max_steps: int = 5):
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=1):
        ref = CpuReference(sysm, params, replicas)
        t0 = time.perf_counter()
        steps = 0
        while steps < max_steps and (steps == 0 or time.perf_counter() - t0 < max_seconds):
            ref.step()
            steps += 1
        dt = time.perf_counter() - t0
    return {"value": ns_per_day(replicas * steps, dt), "unit": UNIT, "cores": ref.cores,
            "kind": "port",
            "sample": f"{replicas} replicas x {steps} full MD steps of coil-269 "
                      f"({dt:.1f} s; oracle port of the reference, numpy {np.__version__}, "
                      f"{ref.cores} worker threads x 1 BLAS thread)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits

    sysm, params = workload(args.config, args.system, args.beads, args.cutoff)
    cores = os.cpu_count() or 1
    R = min(args.replicas, max(8, cores))
    with threadpool_limits(limits=1):
        ref = CpuReference(sysm, params, R)
        for _ in range(args.warmup):
            ref.step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ref.step()
        dt = time.perf_counter() - t0
    value = ns_per_day(R * args.steps, dt)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "coil-269 (1ENH stand-in) x replicas, reference CPU "
                                   "algorithm (oracle port)", "replicas_sampled": R,
                       "weights": "init_params(ModelConfig(), 0)" + (
                           " + quantize_model" if args.config == "w16" else "")},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{R} replicas per step on {cores} threads (the metric "
                                       f"is per replica-step; 64-replica workload sampled)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
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
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2602_13140_b200 import _lib
    from paper_2602_13140_b200.engine import MDEngine

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

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

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            g.replay()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        sampler = ClockSampler(vis.split(",")[local] if vis else str(local))
        t_wall = time.perf_counter()
        for s0, s1 in evs:
            if not args.no_flush:
                flush.zero_()
            s0.record(stream)
            g.replay()
            s1.record(stream)
        torch.cuda.synchronize(dev)
        t_wall = time.perf_counter() - t_wall
        clocks = sampler.stop()
        if world > 1:
            dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    peak_mem = torch.cuda.max_memory_allocated(dev)
    flags = eng.flags()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = ns_per_day(R * world * args.steps, ms_max / 1e3)

    # ---- end-to-end through the host-buffer API --------------------------
    hstate = torch.empty((2, R, N, 3), dtype=torch.float32).pin_memory()  # positions, velocities
    hen = torch.empty((2, R), dtype=torch.float32).pin_memory()            # potential, prior
    hstate.copy_(eng.state)
    with torch.cuda.stream(stream):
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            eng.state.copy_(hstate, non_blocking=True)
            eng.run(1, graph_steps=1)  # the public stepping call (graph replay)
            hstate.copy_(eng.state, non_blocking=True)
            hen.copy_(eng.energies, non_blocking=True)
            stream.synchronize()
        e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = ns_per_day(R * world * args.e2e_steps, float(t.item()))
    h2d = 2 * R * N * 3 * 4
    d2h = 2 * R * N * 3 * 4 + 2 * R * 4

    # ---- per-kernel device times (built-in profiler, eager steps) ---------
    lib = _lib.load()
    lib.fcg_profile_enable(1)
    with torch.cuda.stream(stream):
        for _ in range(args.profile_steps):
            eng._md_step()
    prof = _lib.profile_read()
    lib.fcg_profile_enable(0)
    E_tot = eng.flags()["edges"]
    flags = eng.flags()
    per_step_launch = graph_kernel_nodes(g)
    if per_step_launch is None:  # estimate from the profiler's launch brackets
        per_step_launch = sum(c for _, c in prof.values()) / args.profile_steps
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dom_name, (dom_ms, dom_n) = dom
    avg_ms = dom_ms / dom_n
    pk, pk_kind = peaks()
    if dom_name in ("edge_fwd", "edge_bwd"):
        alg = flags["edges"] * flops_per_edge_block()
        achieved = alg / (avg_ms / 1e3) / 1e12
        roof = {"kernel": dom_name, "bound": "tensor", "achieved": achieved,
                "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s",
                "frac": achieved / pk["bf16_tflops_sustained"],
                "peak_kind": f"{pk_kind} bf16 sustained (MEASURED_PEAKS.json)",
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
    if ncu.exists():
        try:
            roof["traffic"] = json.loads(ncu.read_text()).get(dom_name, {}).get("dram_bytes")
        except Exception:
            pass
    share = {k: round(v[0] / sum(x[0] for x in prof.values()), 4) for k, v in prof.items()}

    # ---- end-of-run gather of per-replica observables (NCCL) -------------
    energies = eng.potential.clone()
    if world > 1:
        from paper_2602_13140_b200.sharding import gather_replicas
        energies = gather_replicas(energies, R * world)

    if rank == 0:
        sysline = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                   "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                   "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                   "dtype": "f32" if args.config == "fp32" else "f16-weights/f32-accum",
                   "data": "synthetic (generate_system coil-269 seed 0; random-init weights)",
                   "config": {"workload": (f"1ENH stand-in coil-269, {R} replicas/GPU, T=3 D=128 "
                                           f"D_r=64 r_cut={args.cutoff} nm, dt=4 fs, nbr rebuild "
                                           "every step") if (args.system, args.beads) == ("coil", 269)
                              else (f"{args.system}-{args.beads} (BASELINE configs[4] sweep), "
                                    f"{R} replicas/GPU, r_cut={args.cutoff} nm, dt=4 fs"),
                              "replicas_per_gpu": R, "total_replicas": R * world,
                              "weights": args.config, "parallelism": f"replica-shard x{world}",
                              "l2": "flushed (256 MiB write) before every timed step"
                                    if not args.no_flush else "not flushed",
                              "mean_edges_per_replica": E_tot / R},
                   "gpu_launches": int(round(per_step_launch * args.steps)),
                   "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                           "d2h_bytes_per_step": d2h, "steps": args.e2e_steps},
                   "roofline": roof, "clocks": clocks,
                   "kernel_share": share,
                   "peak_mem_bytes": int(peak_mem),
                   "flags": {k: flags[k] for k in ("overflow", "blowup", "max_degree")},
                   "energy_mean": float(energies.double().mean().item())}
        if world == 1 and not args.no_gpu_baseline:
            from paper_2602_13140_b200.ablation import compare_on_engine
            sysline["gpu_materialized_baseline"] = compare_on_engine(eng, params)
        if world == 1 and not args.no_cpu_baseline:
            sysline["cpu_baseline"] = cpu_baseline(sysm, params, R)
        print(json.dumps(sysline), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
