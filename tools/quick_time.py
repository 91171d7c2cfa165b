"""Quick device timing of the ID/FD kernels per strategy (development aid, not the bench)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402


def time_call(fn, reps=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    cases = [("C3", torch.float64), ("C3", torch.float32), ("C2", torch.float64), ("C2", torch.float32)]
    for name, dt in cases:
        cfg = synth.CONFIGS[name]
        n, B = cfg["n"], cfg["batch"]
        q, qd, qdd = synth.states(cfg["seed"], n, 0, B, cfg["ranges"])
        tq, tqd, tqdd = (torch.from_numpy(x).to("cuda", dt) for x in (q, qd, qdd))
        model = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"])
        out = torch.empty_like(tq)
        for strat in ("thread", "generic", "warp_scan"):
            model.set_strategy(strat)
            ms = time_call(lambda: rd.inverse_dynamics(model, tq, tqd, tqdd, out))
            flops = (379 * n - 96) * B
            print(f"{name} {str(dt)[6:]} {strat:8s} n={n} B={B}: {ms:.4f} ms  {B / ms * 1e3:.3e} evals/s  "
                  f"{flops / ms / 1e9:.2f} TFLOP/s (lean)", flush=True)
    # small-batch latency sweep (paper's group-number axis)
    cfg = synth.CONFIGS["C3"]
    model = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"])
    for B in (1, 32, 1000, 10000, 100000):
        q, qd, qdd = synth.states(cfg["seed"], 30, 0, B)
        tq, tqd, tqdd = (torch.from_numpy(x).cuda() for x in (q, qd, qdd))
        out = torch.empty_like(tq)
        res = []
        for strat in ("thread", "warp_scan", "generic"):
            model.set_strategy(strat)
            res.append(f"{strat}={time_call(lambda: rd.inverse_dynamics(model, tq, tqd, tqdd, out)) * 1e3:.1f}us")
        print(f"C3-robot B={B}: " + " ".join(res), flush=True)
    cfg = synth.CONFIGS["C4"]
    n, B = cfg["n"], cfg["batch"]
    q, qd, qdd = synth.states(cfg["seed"], n, 0, B)
    tq, tqd, tt = (torch.from_numpy(x).to("cuda") for x in (q, qd, qdd))
    model = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"])
    out = torch.empty_like(tq)
    ms = time_call(lambda: rd.forward_dynamics(model, tq, tqd, tt, out), reps=10, warm=2)
    print(f"C4 FD aba n={n} B={B}: {ms:.4f} ms {B / ms * 1e3:.3e} evals/s "
          f"{(928 * n - 599) * B / ms / 1e9:.2f} TFLOP/s (lean)", flush=True)


if __name__ == "__main__":
    main()
