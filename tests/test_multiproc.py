"""World-size-2 gloo tests (CPU) of the multi-GPU host logic:
shard ranges partition the batch, per-rank regenerated inputs equal the slices
of the full batch bit-for-bit, the gather reassembles tau in order, and the
MAX-over-ranks timing reduction works.  The per-shard compute here is the CPU
oracle standing in for the GPU kernel (no GPU in this container)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_1609_04493_b200.sharding import shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions():
    for total in (0, 1, 7, 1000, 1_000_003):
        for world in (1, 2, 3, 8):
            rs = [shard_range(total, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            for (a0, a1), (b0, b1) in zip(rs, rs[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, total, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1609_04493_b200.sharding import gather_rows
    cfg = synth.CONFIGS["C3"]
    robot = synth.random_chain(6, 1006)
    b0, b1 = shard_range(total, world, rank)
    q, qd, qdd = synth.states(cfg["seed"], 6, b0, b1)             # regenerated from global indices
    tau = oracle.rnea_batch(robot, cfg["gravity"], q, qd, qdd, nthreads=1)
    full = gather_rows(torch.from_numpy(tau), total)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)                      # bench.py's timing reduction
    if rank == 0:
        np.save(os.path.join(out_dir, "full.npy"), full.numpy())
        np.save(os.path.join(out_dir, "tmax.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [1001, 64])
def test_two_rank_shard_gather_matches_single(tmp_path, total):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), total, str(tmp_path)), nprocs=world, join=True)
    import oracle
    cfg = synth.CONFIGS["C3"]
    robot = synth.random_chain(6, 1006)
    q, qd, qdd = synth.states(cfg["seed"], 6, 0, total)
    ref = oracle.rnea_batch(robot, cfg["gravity"], q, qd, qdd, nthreads=1)
    full = np.load(tmp_path / "full.npy")
    np.testing.assert_array_equal(full, ref)                      # bit-identical across sharding
    assert np.load(tmp_path / "tmax.npy")[0] == 2.0


def test_states_are_shard_invariant():
    full = synth.states(5, 30, 0, 5000)
    for a, b in [(0, 1234), (1234, 3000), (3000, 5000)]:
        part = synth.states(5, 30, a, b)
        for x, y in zip(full, part):
            np.testing.assert_array_equal(x[:, a:b], y)
