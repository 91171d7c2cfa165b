"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Each strategy / FD algorithm on small ragged batches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402

for dt in (torch.float64, torch.float32):
    for n, pf in ((7, 0.0), (30, 0.0), (12, 0.4), (40, 0.0), (25, 0.0)):
        robot = synth.random_chain(n, 50 + n, prismatic_fraction=pf)
        model = rd.Model.from_robot(robot, synth.GRAVITY_Z)
        for B in (1, 37, 300):
            q, qd, qdd = (torch.from_numpy(x).to("cuda", dt) for x in synth.states(1, n, 0, B))
            skip = os.environ.get("SKIP_STRATS", "").split(",")
            # SKIP_STASH=1: leave out THREAD only where it runs the TMEM stash kernel
            # (synccheck cannot run tcgen05.alloc, profiles/r02/sanitizer/README.md)
            stash = (n > 12) if dt == torch.float64 else (n in (25, 26) or n > 32)
            if os.environ.get("SKIP_STASH") == "1" and stash:
                skip = skip + ["thread"]
            for strat in ("thread", "warp_scan", "generic", "reverse", "block_scan", "warp_scan_eq13",
                          "warp_scan_eq15", "chunk:2", "chunk:4", "chunk:8", "chunk:32"):
                if strat.split(":")[0] in skip:
                    continue
                model.set_strategy(strat)
                rd.inverse_dynamics(model, q, qd, qdd)
            tau = rd.inverse_dynamics(model, q, qd, qdd)
            bnd = tuple(torch.ones((6, B), dtype=dt, device="cuda") * 0.1 for _ in range(3))
            for strat in ("thread", "warp_scan", "generic", "reverse"):
                if strat in skip:
                    continue
                model.set_strategy(strat)
                rd.inverse_dynamics(model, q, qd, qdd, boundary=bnd)
            model.set_strategy("auto")
            model.set_fd_algo("aba")
            rd.forward_dynamics(model, q, qd, tau, boundary=bnd)
            for algo in ("aba", "jsiia", "aba_scan", "aba_merged"):
                if (algo == "aba_merged" and n > 31) or (algo in ("jsiia", "aba_scan") and n > 256):
                    continue
                model.set_fd_algo(algo)
                rd.forward_dynamics(model, q, qd, tau)
                st = torch.empty(B, dtype=torch.int32, device="cuda")
                rd.forward_dynamics(model, q, qd, tau, status=st)
torch.cuda.synchronize()
print("sanitize_run ok")
