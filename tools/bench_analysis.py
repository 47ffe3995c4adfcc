"""Throughput of the GPU trajectory analysis against
the reference's CPU algorithm (the oracle port, same numpy calls).

    python tools/bench_analysis.py [frames=6400] [beads=269] [cpu_sample=8]

Frames: the coil native structure with Gaussian noise (amplitude cycling
0.02-0.5 nm) under random rigid motions — 64 replicas x 100 output frames
by default.  Prints one JSON line: frames/s per metric on the GPU (device
time with CUDA events around the launches, inputs resident; and end to end
from host arrays), and the CPU oracle's frames/s on a bounded sample.
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from oracle import analysis_oracle as AO  # noqa: E402  (CPU baseline only)
from paper_2602_13140_b200 import _lib  # noqa: E402
from paper_2602_13140_b200 import analysis as A  # noqa: E402
from paper_2602_13140_b200.inputs import generate_system  # noqa: E402


def frames_for(native, F, rng):
    amps = np.array([0.02, 0.05, 0.1, 0.2, 0.5])[np.arange(F) % 5]
    x = native[None] + amps[:, None, None] * rng.standard_normal((F,) + native.shape)
    out = np.empty_like(x)
    for f in range(F):
        q, r = np.linalg.qr(rng.standard_normal((3, 3)))
        q *= np.sign(np.diag(r))
        if np.linalg.det(q) < 0:
            q[:, 0] = -q[:, 0]
        out[f] = x[f] @ q.T + rng.standard_normal(3)
    return out


def main():
    F = int(sys.argv[1]) if len(sys.argv) > 1 else 6400
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 269
    sample = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    rng = np.random.default_rng(0)
    native = generate_system("coil", n, 0).positions.astype(np.float64)
    frames = frames_for(native, F, rng)
    cs = A.build_contacts(native)
    lib = _lib.load()
    v = _lib.vp
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    dx = torch.as_tensor(frames).cuda()
    dy = torch.as_tensor(native).cuda()
    win = A.gdt_windows(n)
    dwin = torch.as_tensor(win).cuda()
    cut = (C.c_double * 4)(*A.GDT_CUTOFFS_NM)
    best = torch.empty(F, 4, dtype=torch.int32, device="cuda")
    rms = torch.empty(F, dtype=torch.float64, device="cuda")
    deg = torch.empty(F, dtype=torch.int32, device="cuda")
    pairs = torch.as_tensor(cs.pairs.astype(np.int32)).cuda()
    r0 = torch.as_tensor(cs.ref_dist).cuda()
    q = torch.empty(F, dtype=torch.float64, device="cuda")
    calls = {
        "gdt_ts": lambda: lib.fcg_gdt_counts(v(dx), v(dy), F, n, v(dwin), len(win),
                                             C.cast(cut, C.c_void_p), v(best), s),
        "rmsd": lambda: lib.fcg_kabsch(v(dx), v(dy), F, n, v(rms), None, None, v(deg), s),
        "q": lambda: lib.fcg_native_q(v(dx), F, n, v(pairs), v(r0), cs.count, A.CONTACT_BETA,
                                      A.CONTACT_LAMBDA, v(q), s),
    }
    dev = {}
    for name, fn in calls.items():
        for _ in range(2):
            _lib.check(fn(), name)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        dev[name] = e0.elapsed_time(e1) / reps / 1e3
    # end to end through the public API from host arrays (incl. graph_stats)
    t0 = time.perf_counter()
    m = A.compute_metrics([(k, 0, None, f) for k, f in enumerate(frames)], native, 1.5,
                          contacts=cs, with_gdt=True)
    e2e = time.perf_counter() - t0
    # CPU: the reference's algorithm (oracle port) on a bounded sample
    idx = np.linspace(0, F - 1, sample).astype(int)
    t0 = time.perf_counter()
    cpu_gdt = [AO.gdt_ts(frames[i], native) for i in idx]
    t_gdt = (time.perf_counter() - t0) / sample
    t0 = time.perf_counter()
    for i in idx:
        AO.kabsch(frames[i], native)
        AO.native_q(frames[i], cs.pairs, cs.ref_dist)
    t_rq = (time.perf_counter() - t0) / sample
    assert np.array_equal(np.asarray(cpu_gdt), m.gdt[idx]), "GDT-TS mismatch vs the oracle"
    # fp64 work of the GDT search: per seed ~ (21 L + 30 n) flop + the eigen solves
    print(json.dumps({
        "workload": f"coil-{n} native vs {F} perturbed frames (64 replicas x {F // 64} frames)",
        "gdt_seeds_per_frame": int(len(win)),
        "gpu_frames_per_s": {k: F / t for k, t in dev.items()},
        "gpu_ms": {k: 1e3 * t for k, t in dev.items()},
        "e2e_compute_metrics_frames_per_s": F / e2e,
        "e2e_compute_metrics_s": e2e,
        "cpu_frames_per_s": {"gdt_ts": 1.0 / t_gdt, "rmsd+q": 1.0 / t_rq},
        "cpu_sample": f"{sample} frames, 1 thread (oracle port of analysis.py)",
        "gdt_speedup_device": t_gdt * F / dev["gdt_ts"],
    }))


if __name__ == "__main__":
    main()
