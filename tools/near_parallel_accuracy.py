"""fp64 accuracy of the DH-frame kernels on chains whose consecutive joint axes are NEARLY
parallel (a calibrated planar / UR-like arm: each axis tilted by eps), against the oracle
and the joint-frame GENERIC kernel.  Development aid."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import oracle, synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import dh_conditioning as dhc  # noqa: E402

g = synth.GRAVITY_Z
dev = lambda x: torch.from_numpy(x).cuda()  # noqa: E731


print("n,eps,stretch,strategy,max_rel_err,resolved")
for n in (6, 30):
    for eps in (0.0, 3e-2, 1e-2, 3e-3, 1e-3, 3e-4, 1e-4):
        r = synth.tilted_planar(n, eps, 5 + n)
        q, qd, qdd = synth.states(37, n, 0, 256)
        ref = oracle.rnea_batch(r, g, q, qd, qdd)
        m = rd.Model.from_robot(r, g)
        for s in ("thread", "reverse", "generic", "auto"):
            m.set_strategy(s)
            tau = rd.inverse_dynamics(m, dev(q), dev(qd), dev(qdd)).cpu().numpy()
            err = (np.abs(tau - ref).max(axis=0) / np.abs(ref).max(axis=0)).max()
            print(f"{n},{eps:g},{dhc.stretch(r):.3g},{s},{err:.3e},{m.resolve_strategy(256, True)}", flush=True)
