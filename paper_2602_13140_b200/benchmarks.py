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


def measure_peak_alloc(params, positions, types, r_cut: float) -> dict:
    """Peak device memory above the live allocations of one energy+forces
    evaluation per schedule (the reference's AllocTracker, traffic.py:185-214,
    measured instead of modelled)."""
    from .ablation import TorchModel, materialized_energy_forces
    from .csr import device_csr
    from .schnet import PipelineMode, flash_energy_forces
    torch = _torch()
    pos = np.asarray(positions, np.float32)
    out = {}
    flash_energy_forces(pos, types, params, PipelineMode())  # persistent buffers first
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    flash_energy_forces(pos, types, params, PipelineMode())
    torch.cuda.synchronize()
    out["flash_peak"] = int(torch.cuda.max_memory_allocated() - base)
    p, nbr, _rev, own = (torch.as_tensor(a).cuda() for a in device_csr(pos, r_cut))
    model = TorchModel(params, torch.float32)
    dpos = torch.as_tensor(pos).cuda()
    dtyp = torch.as_tensor(np.asarray(types).astype(np.int64)).cuda()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    materialized_energy_forces(model, dpos, dtyp, p, nbr, own, 1, pos.shape[0], False)
    torch.cuda.synchronize()
    out["reference_peak"] = int(torch.cuda.max_memory_allocated() - base)
    out["ratio"] = out["reference_peak"] / max(out["flash_peak"], 1)
    return out


def run_bench(params, system, rc_sim: dict, replica_counts, combos, steps: int = 5,
              seed: int = 0) -> list[dict]:
    """Replica counts x backend flags sweep (bench.py:121-192): each cell is
    a short run_simulation; throughput next to the modelled IO of both
    pipelines at the observed mean edge count; speed-up relative to the
    all-off (materialising + scatter) cell at the same replica count.  As in
    the reference, the quant flag is carried but does not change the run."""
    from .langevin import SimConfig, run_simulation, throughput_report
    from .schnet import PipelineMode, io_model_base, io_model_flash
    rows, reference_rate = [], {}
    for replicas in replica_counts:
        for fused, segred, quant in combos:
            sim = SimConfig(dt_fs=rc_sim.get("dt_fs", 4.0),
                            temperature=rc_sim.get("temperature", 300.0),
                            friction=rc_sim.get("friction", 1.0), n_steps=steps,
                            n_replicas=replicas, seed=seed,
                            neighbor_stride=rc_sim.get("neighbor_stride", 1),
                            output_stride=max(steps, 1), mode="32bit",
                            backend=PipelineMode(fused=fused, segred=segred, quant=quant),
                            workers=rc_sim.get("workers", 1))
            result = run_simulation(params, system, sim, rc_sim["out"])
            rate = throughput_report(result)
            n = system.n_beads
            e_mean = int(round(result.mean_edges))
            cfg = params.config
            io_b = io_model_base(n, e_mean, cfg.hidden_dim, cfg.rbf_dim, cfg.num_blocks, 4)
            io_f = io_model_flash(n, e_mean, cfg.hidden_dim, cfg.rbf_dim, cfg.num_blocks, 4)
            alloc = measure_peak_alloc(params, system.initial_positions(), system.types,
                                       cfg.cutoff)
            if not fused and not segred and not quant:
                reference_rate[replicas] = rate["timestep_mol_per_s"]
            speedup = rate["timestep_mol_per_s"] / reference_rate.get(
                replicas, rate["timestep_mol_per_s"])
            rows.append({
                "system": rc_sim.get("name", "system"), "N": n, "E": e_mean,
                "replicas": replicas, "fused": "on" if fused else "off",
                "segred": "on" if segred else "off", "quant": "on" if quant else "off",
                "steps": steps, "ms_per_step": 1e3 * result.wall_seconds / max(steps, 1),
                "timestep_mol_per_s": rate["timestep_mol_per_s"],
                "ns_per_day": rate["ns_per_day"], "io_base_bytes": io_b,
                "io_flash_bytes": io_f, "io_ratio": io_b / io_f,
                "peak_edge_alloc_bytes": alloc["flash_peak" if fused else "reference_peak"],
                "speedup_vs_reference": speedup})
    return rows


def write_bench_csv(rows: list[dict], path) -> None:
    """bench.py:176-192 format: versioned header, schema line, %.6g floats."""
    cols = BENCH_SCHEMA.split(",")
    with open(path, "w") as f:
        f.write("# flashcg-bench v1\n")
        f.write(BENCH_SCHEMA + "\n")
        for row in rows:
            f.write(",".join(_fmt(row[c]) for c in cols) + "\n")


def _fmt(v) -> str:
    return f"{v:.6g}" if isinstance(v, float) else str(v)
