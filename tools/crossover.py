"""Strategy crossover sweep for the AUTO table: ms per call vs B for thread / reverse /
warp_scan at several n, fp64 and fp32 (device inputs, CUDA events, median)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402
from quick_time import time_call  # noqa: E402

print("dtype,n,B,strategy,ms")
gen = torch.Generator(device="cuda").manual_seed(7)
for dt in (torch.float64, torch.float32):
    for n in (7, 10, 20, 30):
        model = rd.Model.from_robot(synth.random_chain(n, 1000 + n), synth.GRAVITY_Z)
        for B in (2048, 4096, 8192, 16384, 32768, 65536, 131072, 262144):
            q, qd, qdd = (torch.rand((n, B), generator=gen, device="cuda", dtype=torch.float64).to(dt) for _ in range(3))
            out = torch.empty_like(q)
            for strat in ("thread", "reverse", "warp_scan"):
                model.set_strategy(strat)
                if model.resolve_strategy(B, dt == torch.float64) != strat:
                    continue
                ms = time_call(lambda: rd.inverse_dynamics(model, q, qd, qdd, out), reps=30)
                print(f"{'f64' if dt == torch.float64 else 'f32'},{n},{B},{strat},{ms:.5f}", flush=True)
