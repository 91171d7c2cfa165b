"""Device time (graph replay) of GENERIC vs joint-frame REVERSE vs WARP_SCAN on models without a
DH form (screw joints; a nominally planar arm with tilted axes).  Development aid."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402
from grid_time import graph_time  # noqa: E402


def screw_chain(n, seed):
    r = synth.random_chain(n, seed, prismatic_fraction=0.0)
    for i in range(0, n, 3):
        r["S"][i, :3] += 0.15 * r["S"][i, 3:]
    return r


print("robot,n,B,dtype,strategy,ms,auto")
for name, n, r in (("tilted", 6, synth.tilted_planar(6, 1e-3, 11)), ("screw", 7, screw_chain(7, 907)),
                   ("screw", 12, screw_chain(12, 912)), ("tilted", 30, synth.tilted_planar(30, 1e-3, 35))):
    m = rd.Model.from_robot(r, synth.GRAVITY_Z)
    for dt in (torch.float64, torch.float32):
        for B in (4096, 16384, 100000, 1000000):
            tq, tqd, tqdd = synth.states_device(3, n, 0, B, dtype=dt)
            out = torch.empty_like(tq)
            for s in ("generic", "reverse", "warp_scan", "thread", "auto"):
                if s == "warp_scan" and (n > 32 or B > 100000):
                    continue
                m.set_strategy(s)
                ms = graph_time(lambda st=None: rd.inverse_dynamics(m, tq, tqd, tqdd, out, stream=st), reps=10)
                print(f"{name},{n},{B},{str(dt)[6:]},{s},{ms:.4f},{m.resolve_strategy(B, dt == torch.float64)}", flush=True)
