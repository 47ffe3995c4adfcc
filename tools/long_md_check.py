"""Long-run stability and thermostat check of the GPU MD step: coil-269 x 64
replicas (the C2 workload), BAOAB at 300 K / 1 ps^-1 / 4 fs, from zero
velocities.  Reports the kinetic temperature per 1000-step block (it must
approach 300 K: equipartition, the reference's test_md.py:117-133 bar is
+-8%), potential/prior energies, edge counts and the blow-up flag.  Writes
one JSON line."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_13140_b200.engine import MDEngine  # noqa: E402
from paper_2602_13140_b200.inputs import generate_system  # noqa: E402
from paper_2602_13140_b200.modelparams import ModelConfig, init_params  # noqa: E402

KB = 0.00831446261815324


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    block = 1000
    sysm = generate_system("coil", 269, 0)
    params = init_params(ModelConfig(), 0)
    R, N = 64, sysm.n_beads
    eng = MDEngine(params, sysm.types, sysm.masses, sysm.prior, R, dt_fs=4.0, temperature=300.0,
                   friction=1.0, seed=0)
    pos = np.repeat(sysm.positions[None], R, axis=0).astype(np.float32)
    eng.load_state(pos, np.zeros_like(pos), 0)
    eng.evaluate()
    m = torch.as_tensor(np.asarray(sysm.masses, np.float64), device="cuda")[None, :, None]
    rows = []
    t0 = time.perf_counter()
    for b in range(steps // block):
        eng.run(block, graph_steps=50)
        v = eng.vel.double()
        ke = 0.5 * (m * v * v).sum(dim=(1, 2))
        temp = (2.0 * ke / (3 * N * KB)).cpu().numpy()
        fl = eng.flags()
        rows.append({"step": (b + 1) * block, "T_mean": float(temp.mean()),
                     "T_min": float(temp.min()), "T_max": float(temp.max()),
                     "potential_mean": float(eng.potential.double().mean().item()),
                     "prior_mean": float(eng.prior_e.double().mean().item()),
                     "edges_per_replica": fl["edges"] / R, "blowup": fl["blowup"]})
    wall = time.perf_counter() - t0
    late = [r["T_mean"] for r in rows[len(rows) // 2:]]
    print(json.dumps({"steps": steps, "replicas": R, "wall_s": wall,
                      "ns_per_day_incl_host_reads": R * steps * 4e-6 * 86400 / wall,
                      "T_second_half_mean": float(np.mean(late)),
                      "blowup": any(r["blowup"] for r in rows), "blocks": rows}))


if __name__ == "__main__":
    main()
