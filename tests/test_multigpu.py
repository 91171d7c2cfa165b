"""Multi-GPU readiness on one GPU.

* the device state generator (synth/gen.cu) is bit-identical to the numpy one,
  so every rank can generate its shard on its GPU from the GLOBAL indices;
* two ranks (gloo, both on the visible GPU) computing their shards through the
  C ABI and gathering tau give exactly the one-rank tau (bit for bit);
* bench.py's multi-rank path (shard ranges, barrier, MAX all-reduce, gather)
  runs end to end under torchrun with --backend gloo.
The NCCL launch on 8 GPUs uses the same code with backend "nccl"."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synth
from paper_1609_04493_b200.sharding import shard_range

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1609_04493_b200 as rd
    rd.lib()
    return rd


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("seed,n,b0,b1,ranges", [(3, 30, 0, 100_003, "default"), (1, 2, 5, 1005, "C1"),
                                                  (5, 30, 9_999_000, 10_000_000, "default"),
                                                  (4, 100, 2 ** 33 + 7, 2 ** 33 + 5000, "default")])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_device_generator_bit_identical(rd, seed, n, b0, b1, ranges, dtype):
    dt = torch.float64 if dtype == "f64" else torch.float32
    got = synth.states_device(seed, n, b0, b1, ranges, dtype=dt)
    want = synth.states(seed, n, b0, b1, ranges)
    for g, w in zip(got, want):
        assert g.dtype == dt and tuple(g.shape) == w.shape
        assert torch.equal(g.cpu(), torch.from_numpy(w).to(dt))


def _rank_worker(rank, world, port, total, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import paper_1609_04493_b200 as rd
    from paper_1609_04493_b200.sharding import gather_rows
    torch.cuda.set_device(0)                               # both ranks share the one GPU
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.CONFIGS["C3"]
    b0, b1 = shard_range(total, world, rank)
    q, qd, qdd = synth.states_device(cfg["seed"], 30, b0, b1)      # the shard, generated on device
    model = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"])
    tau = rd.inverse_dynamics(model, q, qd, qdd)
    full = gather_rows(tau.cpu(), total)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_equal_one_rank_bit_for_bit(rd, tmp_path):
    import torch.multiprocessing as mp
    total = 300_001                       # ragged: 150,001 + 150,000 states, THREAD on every shard
    out = str(tmp_path / "tau2.npy")
    mp.spawn(_rank_worker, args=(2, _free_port(), total, out), nprocs=2, join=True)
    cfg = synth.CONFIGS["C3"]
    model = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"])
    for b0, b1 in (shard_range(total, 2, 0), shard_range(total, 2, 1), (0, total)):
        assert model.resolve_strategy(b1 - b0, True) == "thread"
    q, qd, qdd = synth.states_device(cfg["seed"], 30, 0, total)
    one = rd.inverse_dynamics(model, q, qd, qdd).cpu().numpy()
    np.testing.assert_array_equal(np.load(out), one)


def test_bench_multirank_path_gloo(rd):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--backend", "gloo", "--steps", "3", "--warmup", "3", "--batch", "65536",
           "--no-cpu-baseline", "--e2e-steps", "1", "--gather", "--check-gather"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["global_batch"] == 2 * 65536
    assert line["config"]["gather_ms"] is not None and line["e2e"]["value"] > 0
