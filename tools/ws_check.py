"""Parity + timing of one library build's THREAD strategy against the CPU oracle (development aid).

python tools/ws_check.py LIB.so [--n 8,16,21,22,30,32] [--batch 1000,70001,1000000]
Sampled states (every tile boundary neighbourhood + random) compared with oracle.rnea_batch at
the fp64 contract tolerance (1e-10 of max|tau| per link); then CUDA-graph device time at C3."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1609_04493_b200 as rd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("lib")
ap.add_argument("--n", default="8,16,21,22,25,30,32")
ap.add_argument("--batch", default="1000,70001,1000000")
ap.add_argument("--time-n", default="30")
a = ap.parse_args()
rd.LIB_PATH = a.lib
import torch  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402
from grid_time import graph_time  # noqa: E402

g = synth.GRAVITY_Z
worst = 0.0
for n in map(int, a.n.split(",")):
    robot = synth.random_chain(n, 1000 + n)
    m = rd.Model.from_robot(robot, g)
    m.set_strategy("thread")
    for B in map(int, a.batch.split(",")):
        tq, tqd, tqdd = synth.states_device(7, n, 0, B, dtype=torch.float64)
        tau = rd.inverse_dynamics(m, tq, tqd, tqdd).cpu().numpy()
        rng = np.random.default_rng(n * 7 + B)
        idx = set(rng.integers(0, B, size=min(B, 2000)).tolist())
        for t in range(0, B, 256):                      # tile boundaries (256-state tiles)
            if t % (256 * 37) == 0 or t < 256 * 300:
                idx.update(x for x in (t - 1, t, t + 255) if 0 <= x < B)
        idx.update((0, B - 1))
        idx = np.array(sorted(idx))
        q, qd, qdd = (x.cpu().numpy()[:, idx] for x in (tq, tqd, tqdd))
        ref = oracle.rnea_batch(robot, g, q, qd, qdd)
        err = (np.abs(tau[:, idx] - ref).max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1e-300)).max()
        worst = max(worst, err)
        print(f"n={n} B={B} sampled={len(idx)} rel_err={err:.3e} launches={rd.last_launch_count()}", flush=True)
print(f"WORST {worst:.3e} {'OK' if worst <= 1e-10 else 'FAIL'}")
for n in map(int, a.time_n.split(",")):
    robot = synth.random_chain(n, 1000 + n)
    m = rd.Model.from_robot(robot, g)
    m.set_strategy("thread")
    B = 1000000
    tq, tqd, tqdd = synth.states_device(3, n, 0, B, dtype=torch.float64)
    out = torch.empty_like(tq)
    ms = graph_time(lambda s=None: rd.inverse_dynamics(m, tq, tqd, tqdd, out, stream=s), reps=20)
    print(f"TIME n={n} B={B} {ms:.4f} ms frac={(379 * n - 96) * B / ms / 1e9 / 37.22496:.3f}")
