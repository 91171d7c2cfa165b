"""Run one config/strategy a few times (for ncu captures)."""
import argparse, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1609_04493_b200 as rd

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--strategy", default="auto")
ap.add_argument("--dtype", default="f64")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--fd", action="store_true")
ap.add_argument("--lib", default="")
ap.add_argument("--n", type=int, default=0, help="random chain with n links (overrides the config)")
ap.add_argument("--fd-algo", default="aba")
a = ap.parse_args()
if a.lib:
    rd.LIB_PATH = a.lib
cfg = dict(synth.CONFIGS[a.config])
if a.n:
    cfg.update(n=a.n, robot="random")
n = cfg["n"]; B = a.batch or cfg["batch"]
dt = torch.float64 if a.dtype == "f64" else torch.float32
tq, tqd, tqdd = synth.states_device(cfg["seed"], n, 0, B, cfg["ranges"], dtype=dt)
m = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"])
m.set_strategy(a.strategy)
m.set_fd_algo(a.fd_algo)
if a.fd:                                    # consistent torques for the FD run
    tqdd = rd.inverse_dynamics(m, tq, tqd, tqdd).clone()
out = torch.empty_like(tq)
for _ in range(a.reps):
    if a.fd:
        rd.forward_dynamics(m, tq, tqd, tqdd, out)
    else:
        rd.inverse_dynamics(m, tq, tqd, tqdd, out)
torch.cuda.synchronize()
print("done", a)
