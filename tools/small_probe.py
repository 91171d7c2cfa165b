"""Small-batch timing three ways (development aid): per call with the GPU idle
(host call latency included), back-to-back calls (launch throughput), and a
CUDA graph of K calls replayed (device time per call).  CSV to stdout."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def single(fn, reps=50):
    ts = []
    for _ in range(reps):
        a, b = ev(), ev()
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e3


def b2b(fn, k=200):
    a, b = ev(), ev()
    a.record()
    for _ in range(k):
        fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) * 1e3 / k


def graph(fn, k=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(k):
            fn()
    g.replay(); torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = ev(), ev()
        a.record(); g.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e3 / k


def main():
    cfgs = sys.argv[1:] or ["C2"]
    print("config,dtype,B,strategy,single_us,b2b_us,graph_us")
    for name in cfgs:
        cfg = synth.CONFIGS[name]
        n = cfg["n"]
        model = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"])
        for dt in (torch.float64, torch.float32):
            for B in (1, 1000, 10000, 100000):
                q, qd, qdd = (torch.from_numpy(x).to("cuda", dt) for x in synth.states(cfg["seed"], n, 0, B, cfg["ranges"]))
                out = torch.empty_like(q)
                for strat in ("auto", "thread", "reverse", "warp_scan"):
                    model.set_strategy(strat)
                    fn = lambda: rd.inverse_dynamics(model, q, qd, qdd, out)  # noqa: E731
                    for _ in range(5):
                        fn()
                    torch.cuda.synchronize()
                    name_s = model.resolve_strategy(B, dt == torch.float64) if strat == "auto" else strat
                    print(f"{name},{str(dt)[6:]},{B},{strat}:{name_s},{single(fn):.1f},{b2b(fn):.1f},{graph(fn):.1f}",
                          flush=True)


if __name__ == "__main__":
    main()
