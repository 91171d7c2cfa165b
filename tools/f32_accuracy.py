"""fp32 accuracy per strategy (oracle on the fp32-rounded inputs): random chains and the
tilted planar arm.  Development aid."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import oracle, synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402

g = synth.GRAVITY_Z
print("robot,n,strategy,max_rel_err,resolved")
robots = [("random", n, synth.random_chain(n, 1000 + n, prismatic_fraction=0.05)) for n in (7, 30, 100, 200)]
robots += [(f"tilted{eps:g}", 30, synth.tilted_planar(30, eps, 35)) for eps in (3e-2,)]
for name, n, r in robots:
    q, qd, qdd = synth.states(41, n, 0, 512)
    q32, qd32, qdd32 = (x.astype(np.float32) for x in (q, qd, qdd))
    ref = oracle.rnea_batch(r, g, *(x.astype(np.float64) for x in (q32, qd32, qdd32)))
    m = rd.Model.from_robot(r, g)
    for s in ("thread", "reverse", "chunk", "generic", "warp_scan", "block_scan", "auto"):
        if s == "block_scan" and n > 512:
            continue
        m.set_strategy(s)
        tau = rd.inverse_dynamics(m, *(torch.from_numpy(x).cuda() for x in (q32, qd32, qdd32))).cpu().numpy()
        err = (np.abs(tau - ref).max(axis=0) / np.abs(ref).max(axis=0)).max()
        print(f"{name},{n},{s},{err:.3e},{m.resolve_strategy(512, False)}", flush=True)
