"""fp64 error of each ID strategy against the oracle on long chains (n = 100..1000):
max over states of max_i |tau - tau_oracle| / max_i |tau_oracle|.  Development aid."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import oracle, synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402

g = synth.GRAVITY_Z
print("n,strategy,max_rel_err,auto_pick")
for n, seed in ((30, 1030), (100, 1800), (200, 1900), (300, 2000), (400, 2100), (1000, 1700)):
    r = synth.random_chain(n, seed, prismatic_fraction=0.05)
    q, qd, qdd = synth.states(29, n, 0, 97)
    ref = oracle.rnea_batch(r, g, q, qd, qdd)
    m = rd.Model.from_robot(r, g)
    dev = lambda x: torch.from_numpy(x).cuda()  # noqa: E731
    for s in ("thread", "reverse", "chunk", "generic", "block_scan", "warp_scan", "auto"):
        if s == "thread" and n > 32:
            continue
        if s == "block_scan" and n > 512:
            continue
        try:
            m.set_strategy(s)
            tau = rd.inverse_dynamics(m, dev(q), dev(qd), dev(qdd)).cpu().numpy()
        except Exception as e:  # noqa: BLE001
            print(f"{n},{s},unsupported,{e}")
            continue
        err = (np.abs(tau - ref).max(axis=0) / np.abs(ref).max(axis=0)).max()
        print(f"{n},{s},{err:.3e},{m.resolve_strategy(97, True) if s == 'auto' else ''}", flush=True)
