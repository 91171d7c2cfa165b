import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_04493_b200 as rd
if len(sys.argv) > 1:
    rd.LIB_PATH = sys.argv[1]
import torch, numpy as np, synth
from quick_time import time_call
cfg = synth.CONFIGS["C3"]
q, qd, qdd = synth.states(cfg["seed"], 30, 0, 1_000_000)
tq, tqd, tqdd = (torch.from_numpy(x).cuda() for x in (q, qd, qdd))
m = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"]); m.set_strategy("thread")
out = torch.empty_like(tq)
print(rd.LIB_PATH, f"{time_call(lambda: rd.inverse_dynamics(m, tq, tqd, tqdd, out), reps=50):.4f} ms")
