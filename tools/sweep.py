"""Paper-shaped throughput sweep (the B200 analogue of the paper's
Fig. id_10/id_100 and fd_10/fd_200): evals/s vs group count B for
several link counts n, per strategy / FD algorithm, with the CPU oracle's
evals/s (all host cores, bounded sample) beside each n.

Inputs are synthetic; large batches are drawn on the device with a seeded torch
generator (timing only -- parity is covered by tests/).  Device time with CUDA
events, median of reps after warm-up.  Writes CSV to stdout.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1609_04493_b200 as rd  # noqa: E402


def time_call(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def cpu_rate(robot, g, n, fd, seconds=2.0):
    import oracle
    cores = os.cpu_count() or 1
    chunk = max(64, 8192 // max(1, n // 10))
    q, qd, qdd = synth.states(1, n, 0, chunk)
    tau = oracle.rnea_batch(robot, g, q, qd, qdd, nthreads=cores)
    done, t = 0, 0.0
    while t < seconds:
        t0 = time.perf_counter()
        if fd:
            oracle.fd_batch(robot, g, q, qd, tau, nthreads=cores)
        else:
            oracle.rnea_batch(robot, g, q, qd, qdd, nthreads=cores)
        t += time.perf_counter() - t0
        done += chunk
    return done / t, cores


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--id-n", default="10,30,100")
    ap.add_argument("--fd-n", default="10,30,100,200")
    ap.add_argument("--batches", default="1000,10000,100000,1000000,10000000")
    ap.add_argument("--fd-batches", default="1000,10000,100000")
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--cpu-seconds", type=float, default=2.0)
    args = ap.parse_args()
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    g = synth.GRAVITY_Z
    gen = torch.Generator(device="cuda").manual_seed(1609)
    print("mode,algo,n,B,dtype,ms,evals_per_s,lean_tflops,cpu_oracle_evals_per_s,cpu_cores")

    def rnd(n, B, lo, hi):
        return (torch.rand((n, B), generator=gen, device="cuda", dtype=torch.float64) * (hi - lo) + lo).to(dt)

    for n in [int(x) for x in args.id_n.split(",")]:
        robot = synth.random_chain(n, 1000 + n)
        model = rd.Model.from_robot(robot, g)
        cpu, cores = cpu_rate(robot, g, n, False, args.cpu_seconds)
        for B in [int(x) for x in args.batches.split(",")]:
            if 4 * n * B * (8 if dt == torch.float64 else 4) > 100e9:
                continue
            q, qd, qdd = rnd(n, B, -np.pi, np.pi), rnd(n, B, -1, 1), rnd(n, B, -1, 1)
            out = torch.empty_like(q)
            for strat in ("thread", "warp_scan", "warp_scan_eq13", "warp_scan_eq15", "block_scan", "reverse", "generic", "auto"):
                if strat == "warp_scan_eq15" and B > 100_000:
                    continue                                # the literal 28x28 scan: one warp per SM
                model.set_strategy(strat)
                used = model.resolve_strategy(B, dt == torch.float64)
                if strat != "auto" and used != strat:
                    continue
                reps = 20 if B <= 1_000_000 else 5
                ms = time_call(lambda: rd.inverse_dynamics(model, q, qd, qdd, out), reps)
                name = strat if strat != "auto" else f"auto:{used}"
                print(f"ID,{name},{n},{B},{args.dtype},{ms:.5f},{B / ms * 1e3:.4e},"
                      f"{(379 * n - 96) * B / ms / 1e9:.3f},{cpu:.4e},{cores}", flush=True)
            del q, qd, qdd, out
            torch.cuda.empty_cache()
    for n in [int(x) for x in args.fd_n.split(",")]:
        robot = synth.random_chain(n, 1000 + n)
        model = rd.Model.from_robot(robot, g)
        cpu, cores = cpu_rate(robot, g, n, True, args.cpu_seconds)
        for B in [int(x) for x in args.fd_batches.split(",")]:
            q, qd, qdd = rnd(n, B, -np.pi, np.pi), rnd(n, B, -1, 1), rnd(n, B, -1, 1)
            model.set_fd_algo("aba")
            tau = rd.inverse_dynamics(model, q, qd, qdd)
            out = torch.empty_like(q)
            for algo in ("aba", "jsiia", "aba_scan", "aba_merged"):
                if (algo == "aba_merged" and n > 31) or (algo in ("jsiia", "aba_scan") and n > 256):
                    continue
                model.set_fd_algo(algo)
                ms = time_call(lambda: rd.forward_dynamics(model, q, qd, tau, out), 10)
                print(f"FD,{algo},{n},{B},{args.dtype},{ms:.5f},{B / ms * 1e3:.4e},"
                      f"{(928 * n - 599) * B / ms / 1e9:.3f},{cpu:.4e},{cores}", flush=True)


if __name__ == "__main__":
    main()
