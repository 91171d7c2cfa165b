"""Device time per ID call over a grid of (n, B, strategy), as CSV (development aid).

Each point captures R back-to-back calls in one CUDA graph and replays it, so the
number is device time per call without the host call path (small batches are
otherwise host-bound).  Inputs are generated on the device (synth.states_device).

    python tools/grid_time.py --n 7,30,100 --B 1000,10000,100000,1000000 \
        --strategies thread,reverse,chunk:2,chunk:8 --dtype f64
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402


def graph_time(fn, reps=20, replays=5):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn(s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(replays):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="30")
    ap.add_argument("--B", default="1000,10000,100000,1000000")
    ap.add_argument("--strategies", default="thread,reverse,chunk")
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--robot", default="random", help="random | arm7")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    print("dtype,n,B,strategy,resolved,ms,evals_per_s,lean_tflops", flush=True)
    for n in (int(x) for x in args.n.split(",")):
        robot = synth.arm7() if args.robot == "arm7" else synth.random_chain(n, 1000 + n)
        model = rd.Model.from_robot(robot, synth.GRAVITY_Z)
        for B in (int(x) for x in args.B.split(",")):
            tq, tqd, tqdd = synth.states_device(3, n, 0, B, dtype=dt)
            out = torch.empty_like(tq)
            for strat in args.strategies.split(","):
                model.set_strategy(strat)
                resolved = model.resolve_strategy(B, dt == torch.float64)
                reps = max(2, min(args.reps, int(2e7 // max(1, n * B))))
                ms = graph_time(lambda s=None: rd.inverse_dynamics(model, tq, tqd, tqdd, out, stream=s), reps)
                print(f"{args.dtype},{n},{B},{strat},{resolved},{ms:.5f},{B / ms * 1e3:.4e},"
                      f"{(379 * n - 96) * B / ms / 1e9:.3f}", flush=True)
            del tq, tqd, tqdd, out


if __name__ == "__main__":
    main()
