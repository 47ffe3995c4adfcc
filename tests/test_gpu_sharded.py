"""Replica sharding through the real engine: ranks of a
torch.distributed group run disjoint replica blocks of one run_simulation
and meet only at output-chunk boundaries (one integer) and at the end (one
gather).  Two ranks share the one GPU of the test box over gloo (NCCL needs
distinct GPUs); the result must equal the unsharded run bit for bit:
final state, trajectory.xyz bytes, scalars.csv except the wall-clock
column, checkpoints.  bench.py's multi-rank launcher is exercised the same
way."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    from paper_2602_13140_b200.inputs import generate_system
    from paper_2602_13140_b200.modelparams import ModelConfig, init_params
    sysm = generate_system("coil", 40, 3)
    params = init_params(ModelConfig(), 0)
    return sysm, params


def _sim(tmp, R, steps, **kw):
    import paper_2602_13140_b200 as P
    return P.SimConfig(dt_fs=4.0, temperature=300.0, friction=1.0, n_steps=steps, n_replicas=R,
                       seed=4, output_stride=5, **kw)


def _worker(rank, world, port, out, R, steps, chk):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist
    import paper_2602_13140_b200 as P
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sysm, params = _setup()
    kw = dict(checkpoint_path=chk, checkpoint_step=7) if chk else {}
    res = P.run_simulation(params, sysm, _sim(out, R, steps, **kw), out, distributed=True)
    np.savez(Path(out) / f"rank{rank}.npz", pos=res.final_state.positions,
             vel=res.final_state.velocities, mean_edges=res.mean_edges,
             traffic=res.traffic.total_bytes, replicas=res.replicas)
    dist.destroy_process_group()


@pytest.mark.parametrize("R,world", [(5, 2), (4, 2)])
def test_sharded_run_simulation_equals_unsharded(tmp_path, R, world):
    import paper_2602_13140_b200 as P
    steps = 13
    sysm, params = _setup()
    single = P.run_simulation(params, sysm, _sim(tmp_path, R, steps, checkpoint_path=str(
        tmp_path / "single.flcg"), checkpoint_step=7), tmp_path / "single")
    out = tmp_path / "sharded"
    out.mkdir()
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, str(out), R, steps,
                                               str(tmp_path / "sharded.flcg")))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    for r in range(world):
        got = np.load(out / f"rank{r}.npz")
        np.testing.assert_array_equal(got["pos"], single.final_state.positions)
        np.testing.assert_array_equal(got["vel"], single.final_state.velocities)
        assert float(got["mean_edges"]) == single.mean_edges
        assert int(got["traffic"]) == single.traffic.total_bytes
        assert int(got["replicas"]) == R
    assert (out / "trajectory.xyz").read_bytes() == single.trajectory_path.read_bytes()
    strip = lambda p: [ln.rsplit(",", 1)[0] for ln in p.read_text().splitlines()]  # noqa: E731
    assert strip(out / "scalars.csv") == strip(single.scalars_path)
    assert (tmp_path / "sharded.flcg").read_bytes() == (tmp_path / "single.flcg").read_bytes()


def test_bench_launches_ranks_itself():
    """`python bench.py --gpus 2` (no torchrun around it) spawns two ranks;
    here they share the one GPU over gloo (--dist-backend gloo
    --share-gpu), and the line reports both ranks' replicas."""
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3", "--replicas", "4", "--e2e-steps", "2",
                        "--dist-backend", "gloo", "--share-gpu", "--no-cpu-baseline",
                        "--no-gpu-baseline"], capture_output=True, text=True, env=env,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["config"]["total_replicas"] == 8
    assert line["end_of_run_gather"]["replicas"] == 8
