"""Single-robot latency as device time: CUDA-graph replay of K calls (host call
path excluded) vs one call with the GPU idle (host path included).  CSV."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402
from small_probe import single, graph  # noqa: E402

print("n,B,strategy,single_us,graph_us")
for n in (8, 32, 64, 128, 256, 512):
    model = rd.Model.from_robot(synth.random_chain(n, 1000 + n), synth.GRAVITY_Z)
    for B in (1, 64):
        q, qd, qdd = (torch.from_numpy(x).cuda() for x in synth.states(1, n, 0, B))
        out = torch.empty_like(q)
        for strat in ("warp_scan", "block_scan", "reverse"):
            model.set_strategy(strat)
            if model.resolve_strategy(B) != strat:
                continue
            fn = lambda: rd.inverse_dynamics(model, q, qd, qdd, out)  # noqa: E731
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            print(f"{n},{B},{strat},{single(fn):.1f},{graph(fn):.1f}", flush=True)
