"""World-size-2 gloo tests of the multi-GPU host logic (CPU only): replica
sharding with rep_offset-keyed noise plus the end-of-run gather reproduce
an unsharded run of the same replicas bit for bit.  The per-shard compute
stand-in is the CPU oracle (the GPU engine is covered by
test_gpu_parity.py::test_replica_sharding_bit_identical)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_13140_b200.sharding import replica_shard


def test_shard_ranges_cover_all():
    for total in (1, 2, 7, 64, 512, 513):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                first, cnt = replica_shard(total, world, r)
                seen.extend(range(first, first + cnt))
            assert seen == list(range(total))
    with pytest.raises(ValueError):
        replica_shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle import flashcg_oracle as O
    from paper_2602_13140_b200.inputs import generate_system
    from paper_2602_13140_b200.modelparams import ModelConfig, init_params
    from paper_2602_13140_b200.sharding import gather_replicas

    sysm = generate_system("coil", 12, 5)
    params = init_params(ModelConfig(hidden_dim=8, rbf_dim=4, num_blocks=1, cutoff=1.2,
                                     num_atom_types=8, filter_hidden_dim=8,
                                     readout_hidden_dim=4), 9)
    first, cnt = replica_shard(total, world, rank)
    pos0 = np.repeat(sysm.positions[None], cnt, axis=0).astype(np.float32)
    pos, vel, F, pot, pri, _ = O.run_md(params, sysm.types, sysm.masses, sysm.prior, pos0,
                                        np.zeros_like(pos0), 6, seed=23, rep_offset=first)
    allpos = gather_replicas(torch.as_tensor(pos), total)
    allpot = gather_replicas(torch.as_tensor(pot), total)
    if rank == 0:
        out_q.put((allpos.numpy(), allpot.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_run_equals_single_run():
    from oracle import flashcg_oracle as O
    from paper_2602_13140_b200.inputs import generate_system
    from paper_2602_13140_b200.modelparams import ModelConfig, init_params

    total, world = 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    allpos, allpot = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0

    sysm = generate_system("coil", 12, 5)
    params = init_params(ModelConfig(hidden_dim=8, rbf_dim=4, num_blocks=1, cutoff=1.2,
                                     num_atom_types=8, filter_hidden_dim=8,
                                     readout_hidden_dim=4), 9)
    pos0 = np.repeat(sysm.positions[None], total, axis=0).astype(np.float32)
    pos, vel, F, pot, pri, _ = O.run_md(params, sysm.types, sysm.masses, sysm.prior, pos0,
                                        np.zeros_like(pos0), 6, seed=23)
    np.testing.assert_array_equal(allpos, pos)
    np.testing.assert_array_equal(allpot, pot)
