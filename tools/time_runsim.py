"""Wall-clock throughput of run_simulation (the reference-facing API, with
trajectory/scalars output) for coil-269 x R replicas."""
import os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_13140_b200 as P
from paper_2602_13140_b200.inputs import generate_system
from paper_2602_13140_b200.modelparams import ModelConfig, init_params

R = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
stride = int(sys.argv[3]) if len(sys.argv) > 3 else 10
sysm = generate_system("coil", 269, 0)
params = init_params(ModelConfig(), 0)
cfg = P.SimConfig(dt_fs=4.0, temperature=300.0, friction=1.0, n_steps=steps, n_replicas=R,
                  seed=0, output_stride=stride)
with tempfile.TemporaryDirectory() as d:
    P.run_simulation(params, sysm, P.SimConfig(dt_fs=4.0, n_steps=20, n_replicas=R,
                                               output_stride=stride), d)  # warm-up
    t = time.perf_counter()
    res = P.run_simulation(params, sysm, cfg, d)
    wall = time.perf_counter() - t
    size = os.path.getsize(os.path.join(d, "trajectory.xyz"))
rep = P.throughput_report(res)
print(f"run_simulation R={R} steps={steps} output_stride={stride}: {wall:.2f} s, "
      f"{rep['ns_per_day']:.1f} ns/day (result wall {res.wall_seconds:.2f} s), "
      f"trajectory {size / 1e6:.1f} MB")
