"""FD device time: joint-frame ABA (workspace) on models without a DH form vs the DH register ABA
on a DH robot of the same length.  Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402
from grid_time import graph_time  # noqa: E402

print("robot,n,B,dtype,algo,ms")
for name, n, r in [("tilted", k, synth.tilted_planar(k, 1e-3, 11 + k)) for k in (4, 6, 7, 8, 10, 12)]:
    m = rd.Model.from_robot(r, synth.GRAVITY_Z)
    for dt in (torch.float64, torch.float32):
        for B in (4096, 100000, 1000000):
            tq, tqd, tqdd = synth.states_device(3, n, 0, B, dtype=dt)
            tau = rd.inverse_dynamics(m, tq, tqd, tqdd).clone()
            out = torch.empty_like(tq)
            for algo in ("aba",):
                m.set_fd_algo(algo)
                ms = graph_time(lambda st=None: rd.forward_dynamics(m, tq, tqd, tau, out, stream=st), reps=10)
                print(f"{name},{n},{B},{str(dt)[6:]},{algo},{ms:.4f}", flush=True)
