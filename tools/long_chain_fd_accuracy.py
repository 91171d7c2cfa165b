"""fp64 FD accuracy per algorithm on long chains: backward error max|RNEA_oracle(q, qd, qdd_gpu) - tau| / max|tau|
and forward error max|qdd_gpu - qdd_oracle| / max|qdd_oracle| (cond(M)-limited).  Development aid."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import oracle, synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402

g = synth.GRAVITY_Z
dev = lambda x: torch.from_numpy(x).cuda()  # noqa: E731
print("n,algo,backward_err,forward_err")
for n, seed in ((30, 1030), (100, 1100), (200, 1900), (400, 2100)):
    r = synth.random_chain(n, seed, prismatic_fraction=0.05)
    q, qd, qdd = synth.states(31, n, 0, 64)
    tau = oracle.rnea_batch(r, g, q, qd, qdd)
    ref = oracle.fd_batch(r, g, q, qd, tau)
    m = rd.Model.from_robot(r, g)
    for algo in ("aba", "jsiia", "aba_scan"):
        if algo != "aba" and n > 256:
            continue
        m.set_fd_algo(algo)
        out = rd.forward_dynamics(m, dev(q), dev(qd), dev(tau)).cpu().numpy()
        back = oracle.rnea_batch(r, g, q, qd, out)
        be = (np.abs(back - tau).max(axis=0) / np.abs(tau).max(axis=0)).max()
        fe = (np.abs(out - ref).max(axis=0) / np.abs(ref).max(axis=0)).max()
        print(f"{n},{algo},{be:.3e},{fe:.3e}", flush=True)
