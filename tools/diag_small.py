"""Per-case parity errors of the THREAD strategy at short n, for one library build
(development aid): python tools/diag_small.py LIB.so"""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_04493_b200 as rd  # noqa: E402
rd.LIB_PATH = sys.argv[1]
import torch  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402

for dt in (torch.float64, torch.float32):
    for n in range(1, 10):
        out = []
        for pf, seed in ((0.0, 1200 + n), (0.4, 1300 + n)):
            r = synth.random_chain(n, seed, prismatic_fraction=pf)
            m = rd.Model.from_robot(r, synth.GRAVITY_Z)
            m.set_strategy("thread")
            for B in (1, 127, 129, 3001):
                q, qd, qdd = synth.states(21, n, 0, B)
                t = [torch.from_numpy(x).to("cuda", dt) for x in (q, qd, qdd)]
                tau = rd.inverse_dynamics(m, *t).double().cpu().numpy()
                q64, qd64, qdd64 = (x.double().cpu().numpy() for x in t)
                ref = oracle.rnea_batch(r, synth.GRAVITY_Z, q64, qd64, qdd64)
                e = (np.abs(tau - ref).max(axis=0) / np.abs(ref).max(axis=0))
                out.append(f"pf{pf}/B{B}:{e.max():.1e}@{int(e.argmax())}")
        rng = np.random.default_rng(n)
        V0, Vd0, Ft = rng.standard_normal((3, 6))
        r = synth.random_chain(n, 1400 + n, prismatic_fraction=0.3)
        m = rd.Model.from_robot(r, (0, 0, 0))
        m.set_boundary(V0, Vd0, Ft)
        m.set_strategy("thread")
        q, qd, qdd = synth.states(22, n, 0, 500)
        t = [torch.from_numpy(x).to("cuda", dt) for x in (q, qd, qdd)]
        tau = rd.inverse_dynamics(m, *t).double().cpu().numpy()
        q64, qd64, qdd64 = (x.double().cpu().numpy() for x in t)
        ref = np.stack([oracle.rnea(r, q64[:, b], qd64[:, b], qdd64[:, b], V0, Vd0, Ft) for b in range(500)], 1)
        e = (np.abs(tau - ref).max(axis=0) / np.abs(ref).max(axis=0))
        out.append(f"bnd:{e.max():.1e}@{int(e.argmax())} (|ref| there {np.abs(ref[:, e.argmax()]).max():.2e})")
        print(str(dt)[-7:], n, " ".join(out), flush=True)
