"""Single-robot / small-batch latency (paper §V-A): device time per
call vs n for each strategy, B in {1, 16, 256}.  CSV to stdout."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402


def time_call(fn, reps=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)) * 1e3


print("n,B,strategy,us")
for n in (8, 16, 32, 64, 128, 256, 512):
    robot = synth.random_chain(n, 1000 + n)
    model = rd.Model.from_robot(robot, synth.GRAVITY_Z)
    for B in (1, 16, 256, 1024, 4096):
        q, qd, qdd = (torch.from_numpy(x).cuda() for x in synth.states(1, n, 0, B))
        out = torch.empty_like(q)
        for strat in ("thread", "warp_scan", "block_scan", "reverse", "generic"):
            model.set_strategy(strat)
            if model.resolve_strategy(B) != strat:
                continue
            us = time_call(lambda: rd.inverse_dynamics(model, q, qd, qdd, out))
            print(f"{n},{B},{strat},{us:.1f}", flush=True)
