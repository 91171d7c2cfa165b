"""A/B timing of one library build: python tools/fake_time.py LIB.so [--config C3] [--fd] [--strategy thread]
[--dtype f64].  Median CUDA-event time of the call over 50 reps (quick_time.time_call)."""
import argparse
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1609_04493_b200 as rd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("lib")
ap.add_argument("--config", default="C3")
ap.add_argument("--fd", action="store_true")
ap.add_argument("--strategy", default="thread")
ap.add_argument("--fd-algo", default="aba")
ap.add_argument("--dtype", default="f64")
ap.add_argument("--n", type=int, default=0, help="random chain with n links (overrides the config)")
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--graph", action="store_true", help="device time: CUDA-graph replay of 20 calls (grid_time)")
a = ap.parse_args()
rd.LIB_PATH = a.lib
import torch  # noqa: E402
import synth  # noqa: E402
from quick_time import time_call  # noqa: E402

cfg = dict(synth.CONFIGS[a.config])
if a.n:
    cfg.update(n=a.n, robot="random")
if a.batch:
    cfg.update(batch=a.batch)
n = cfg["n"]
dt = torch.float64 if a.dtype == "f64" else torch.float32
tq, tqd, tqdd = synth.states_device(cfg["seed"], n, 0, cfg["batch"], cfg["ranges"], dtype=dt)
m = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"])
m.set_strategy(a.strategy)
m.set_fd_algo(a.fd_algo)
out = torch.empty_like(tq)
if a.graph:
    from grid_time import graph_time
    g = ((lambda s=None: rd.forward_dynamics(m, tq, tqd, tqdd, out, stream=s)) if a.fd else
         (lambda s=None: rd.inverse_dynamics(m, tq, tqd, tqdd, out, stream=s)))
    ms = graph_time(g, reps=20)
else:
    f = (lambda: rd.forward_dynamics(m, tq, tqd, tqdd, out)) if a.fd else (lambda: rd.inverse_dynamics(m, tq, tqd, tqdd, out))
    ms = time_call(f, reps=50)
print(os.path.basename(a.lib), a.config, a.dtype, f"n={n} B={cfg['batch']}", "fd" if a.fd else "id",
      a.strategy if not a.fd else a.fd_algo, "graph" if a.graph else "events", f"{ms:.4f} ms")
