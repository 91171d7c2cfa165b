"""bench.py -- batched RNEA throughput on B200 (BASELINE.json metric).

Default workload (N=1): config C3 -- 30-link random serial chain, 1M states per
GPU, fp64, inverse dynamics through the C ABI (rd_inverse_dynamics_f64).
A step is one pass of the whole hot path (one RNEA over the batch).  Under
torchrun each rank evaluates its own 1M-state shard (weak scaling, no
data-path collective); the timed region is bracketed by barrier +
synchronize and the max over ranks is reported.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--dtype f64]
    python bench.py --impl reference      # the CPU oracle arm (rank 0 only)

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "RNEA evals/s (n=30 links, 1M states) at 1/2/4/8 B200; % of FP64 roofline"
UNIT = "evals/s"
# Nominal FP64 CUDA-core peak from the guide's unit counts and clock:
# 148 SMs x 64 DFMA/clk x 2 flop x 1.965 GHz.
PEAK_F64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
PEAK_F32_TFLOPS = 2 * PEAK_F64_TFLOPS
L2_BYTES = 126 * 2 ** 20


def lean_flops_id(n: int) -> int:
    """SURVEY §8(d) algorithmic flop count of one RNEA (FMA = 2, sincos excluded)."""
    return 379 * n - 96


def lean_flops_fd(n: int) -> int:
    return 928 * n - 599


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                self.reasons |= int(self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        busy = [s for s in self.samples]
        return {
            "sm_mhz": float(statistics.median(busy)) if busy else None,
            "sm_max_mhz": self.max_mhz,
            "samples": len(busy),
            "reasons": [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1],
        }


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_baseline(robot, g, cfg, n, seconds=10.0):
    """The oracle as it stands on all host cores, on a bounded sample of the workload."""
    import oracle
    cores = os.cpu_count() or 1
    chunk = 4096 * cores // 8 if cores >= 8 else 4096
    done, t_total, b0 = 0, 0.0, 0
    oracle.rnea_batch(robot, g, *synth.states(cfg["seed"], n, 0, 64, cfg["ranges"]), nthreads=cores)
    while t_total < seconds and done < 40_000_000:
        q, qd, qdd = synth.states(cfg["seed"], n, b0, b0 + chunk, cfg["ranges"])
        t0 = time.perf_counter()
        oracle.rnea_batch(robot, g, q, qd, qdd, nthreads=cores)
        t_total += time.perf_counter() - t0
        done += chunk
        b0 += chunk
    # single-core figure: one thread on the first chunk, ~1-2 s
    q, qd, qdd = synth.states(cfg["seed"], n, 0, chunk, cfg["ranges"])
    t0 = time.perf_counter()
    oracle.rnea_batch(robot, g, q, qd, qdd, nthreads=1)
    one = chunk / (time.perf_counter() - t0)
    return {"value": done / t_total, "unit": UNIT, "cores": cores, "kind": "oracle", "single_core_value": one,
            "sample": f"first {done} states of the {cfg['name']} workload (n={n}), oracle::rnea "
                      f"(C++ -O2, dense 6x6 Eq. 1-2) on {cores} host threads, {t_total:.1f} s; "
                      f"single_core_value: {chunk} states on 1 thread"}


def cpu_baseline_fd(robot, g, cfg, n, seconds=10.0):
    """The oracle's ABA (Eq. 7-8) on all host cores, on a bounded sample of the FD workload."""
    import oracle
    cores = os.cpu_count() or 1
    chunk = 512 * max(1, cores // 4)
    done, t_total, b0 = 0, 0.0, 0
    while t_total < seconds and done < 2_000_000:
        q, qd, qdd = synth.states(cfg["seed"], n, b0, b0 + chunk, cfg["ranges"])
        tau = oracle.rnea_batch(robot, g, q, qd, qdd, nthreads=cores)
        t0 = time.perf_counter()
        oracle.fd_batch(robot, g, q, qd, tau, nthreads=cores)
        t_total += time.perf_counter() - t0
        done += chunk
        b0 += chunk
    q, qd, qdd = synth.states(cfg["seed"], n, 0, chunk, cfg["ranges"])
    tau = oracle.rnea_batch(robot, g, q, qd, qdd, nthreads=cores)
    t0 = time.perf_counter()
    oracle.fd_batch(robot, g, q, qd, tau, nthreads=1)
    one = chunk / (time.perf_counter() - t0)
    return {"value": done / t_total, "unit": UNIT, "cores": cores, "kind": "oracle", "single_core_value": one,
            "sample": f"first {done} states of the {cfg['name']} FD workload (n={n}), oracle::fd_aba "
                      f"(C++ -O2, Eq. 7-8) on {cores} host threads, {t_total:.1f} s; "
                      f"single_core_value: {chunk} states on 1 thread"}


def load_traffic(cfg_name: str, dtype: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full
    capture (profiles/ncu_traffic.json, tools/ncu_traffic.py) and the capture it came from."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"{cfg_name}_{dtype}"), d.get(f"{cfg_name}_{dtype}_source")
    except Exception:
        return None, None


def run_reference(args):
    """--impl reference: the CPU oracle, timed as it stands (rank 0 only)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    cfg = config_of(args)
    n = cfg["n"]
    robot = robot_of(cfg)
    g = cfg["gravity"]
    cores = os.cpu_count() or 1
    # bounded sample per step: calibrate the oracle's rate, then size each step so the
    # whole --warmup + --steps run takes about --ref-seconds (capped at --ref-sample states)
    fd = args.config == "C4"
    cal = 256 if fd else 2048
    qc, qdc, qddc = synth.states(cfg["seed"], n, 0, cal, cfg["ranges"])
    if fd:
        tc = oracle.rnea_batch(robot, g, qc, qdc, qddc, nthreads=cores)
        run = lambda a, b, c, t: oracle.fd_batch(robot, g, a, b, t, nthreads=cores)  # noqa: E731
    else:
        tc = None
        run = lambda a, b, c, t: oracle.rnea_batch(robot, g, a, b, c, nthreads=cores)  # noqa: E731
    t0 = time.perf_counter()
    run(qc, qdc, qddc, tc)
    rate = cal / max(time.perf_counter() - t0, 1e-6)
    sample = int(min(args.ref_sample, max(256, rate * args.ref_seconds / (args.steps + args.warmup))))
    q, qd, qdd = synth.states(cfg["seed"], n, 0, sample, cfg["ranges"])
    tq = oracle.rnea_batch(robot, g, q, qd, qdd, nthreads=cores) if fd else None
    for _ in range(args.warmup):
        run(q, qd, qdd, tq)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run(q, qd, qdd, tq)
    dt = time.perf_counter() - t0
    value = sample * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{cfg['name']}: n={n} {'FD (ABA)' if fd else 'RNEA'} (bounded sample of {sample} "
                               f"states/step of the workload)",
                   "n": n, "states_per_step": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{sample} states of {args.config} per step, oracle::"
                                   f"{'fd_aba' if fd else 'rnea'} on {cores} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_of(args) -> dict:
    """The BASELINE config, optionally overridden by --n / --seed / --model (then
    config.workload says so: the bench line is no longer the config's)."""
    cfg = dict(synth.CONFIGS[args.config], name=args.config)
    if args.n:
        cfg.update(n=args.n, robot="random", name=f"{args.config}+n={args.n}")
    if args.seed is not None:
        cfg.update(seed=args.seed, name=cfg["name"] + f"+seed={args.seed}")
    if args.model:
        from paper_1609_04493_b200 import model_io
        cfg.update(model=model_io.load_model(args.model), name=cfg["name"] + f"+model={os.path.basename(args.model)}")
        cfg["n"] = cfg["model"]["S"].shape[0]
    return cfg


def robot_of(cfg: dict) -> dict:
    return cfg["model"] if "model" in cfg else synth.robot_for(cfg)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3", choices=list(synth.CONFIGS))
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--strategy", default="auto")
    ap.add_argument("--batch", type=int, default=0, help="states per GPU (default: the config's)")
    ap.add_argument("--n", type=int, default=0, help="links of the random chain (overrides the config's n)")
    ap.add_argument("--seed", type=int, default=None, help="state seed (overrides the config's)")
    ap.add_argument("--model", default=None, help="robot model file (JSON, paper_1609_04493_b200.model_io)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--gather", action="store_true", help="time a final all-gather of tau (off the hot path)")
    ap.add_argument("--check-gather", action="store_true", help="with --gather: check the gathered tau")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: ranks may share one GPU)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=65536)
    ap.add_argument("--ref-seconds", type=float, default=60.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import paper_1609_04493_b200 as rd

    world, rank, local = dist_env()
    # one process per GPU; --backend gloo runs the same multi-rank path with several
    # ranks sharing the visible GPU(s) (a test of the host logic, not a scaling run)
    ndev = torch.cuda.device_count()
    local = local % ndev if args.backend == "gloo" else local
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    coll_dev = "cuda" if args.backend == "nccl" else "cpu"     # where the off-path collectives run
    cfg = config_of(args)
    n = cfg["n"]
    fd = args.config == "C4"
    from paper_1609_04493_b200.sharding import shard_range, gather_rows
    per_gpu = args.batch or cfg["batch"]
    total = per_gpu * world if args.scaling == "weak" else per_gpu
    b0, b1 = shard_range(total, world, rank)       # contiguous global-index shard
    per_gpu = b1 - b0
    robot = robot_of(cfg)
    g = cfg["gravity"]
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    # inputs: a pure function of the GLOBAL state index, generated on this rank's GPU
    # (synth/gen.cu: bit-identical to synth.states, which the CPU oracle side uses)
    tq, tqd, tqdd = synth.states_device(cfg["seed"], n, b0, b1, cfg["ranges"], dtype=dt)
    model = rd.Model.from_robot(robot, g)
    model.set_strategy(args.strategy)
    out = torch.empty_like(tq)
    if fd:
        tau_in = rd.inverse_dynamics(model, tq, tqd, tqdd)     # consistent torques (untimed)
        step = lambda: rd.forward_dynamics(model, tq, tqd, tau_in, out)  # noqa: E731
    else:
        step = lambda: rd.inverse_dynamics(model, tq, tqd, tqdd, out)  # noqa: E731
    in_bytes = 3 * n * per_gpu * tq.element_size()
    l2_note = (f"inputs {in_bytes / 2**20:.0f} MiB > L2 {L2_BYTES / 2**20:.0f} MiB, no flush"
               if in_bytes > 2 * L2_BYTES else "L2 flushed between steps (write of 2x L2)")
    flush_buf = None if in_bytes > 2 * L2_BYTES else torch.empty(2 * L2_BYTES // 4, dtype=torch.float32,
                                                                   device="cuda")

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def allreduce_max(vals):
        """MAX over ranks of a few floats (the timing reduction, off the hot path)."""
        if world == 1:
            return vals
        import torch.distributed as dist
        tt = torch.tensor(vals, device=coll_dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return [float(x) for x in tt]

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches = 0
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clock = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    with clock:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for k in range(args.steps):
            if flush_buf is not None:                  # flushed steps: events around each call
                flush_buf.zero_()
                evs[k][0].record(stream)
            step()
            if flush_buf is not None:
                evs[k][1].record(stream)
            launches += rd.last_launch_count()
        t_end.record(stream)
        torch.cuda.synchronize()
    barrier()
    # inputs larger than L2: the K calls run back to back and the average launch duration
    # is the bracketing events' span / K (per-call event pairs would add their own
    # ~2-5 us record gaps to every step); flushed steps: the per-call event pairs
    kernel_ms = ([a.elapsed_time(b) for a, b in evs] if flush_buf is not None
                 else [t_start.elapsed_time(t_end) / args.steps])
    total_ms = t_start.elapsed_time(t_end) if flush_buf is None else sum(kernel_ms)
    avg_kernel_ms = float(np.mean(kernel_ms))
    total_ms, avg_kernel_ms = allreduce_max([total_ms, avg_kernel_ms])
    units = total * args.steps
    value = units / (total_ms / 1e3)

    # optional final gather of tau to every rank over NCCL, timed separately
    gather_ms = None
    if args.gather and world > 1:
        import torch.distributed as dist
        barrier()
        g0 = time.perf_counter()
        full = gather_rows(out if coll_dev == "cuda" else out.cpu(), total)
        torch.cuda.synchronize()
        if args.check_gather:                         # every rank holds the full tau: compare its own slice
            assert torch.equal(full[:, b0:b1].to(out.device), out), "gathered tau differs from the shard"
        gather_ms = (time.perf_counter() - g0) * 1e3
        del full

    # e2e: through the public host-buffer API (pinned host arrays, H2D + kernel + D2H per step)
    e2e = None
    if args.dtype == "f64" and args.e2e_steps > 0:
        third = tau_in if fd else tqdd                             # FD: the consistent torques
        pq, pqd, pqdd = (x.cpu().pin_memory() for x in (tq, tqd, third))
        pout = torch.empty_like(pq).pin_memory()
        host_api = rd.forward_dynamics_host if fd else rd.inverse_dynamics_host
        host_api(model, pq, pqd, pqdd, pout)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            host_api(model, pq, pqd, pqdd, pout)
        e2e_s = allreduce_max([time.perf_counter() - t0])[0]
        e2e = {"value": total * args.e2e_steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": 3 * n * total * 8, "d2h_bytes_per_step": n * total * 8,
               "api": ("rd_forward_dynamics_host_f64" if fd else "rd_inverse_dynamics_host_f64")
                      + " (pinned host buffers, chunked 2-stream pipeline)"}

    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    flops = (lean_flops_fd(n) if fd else lean_flops_id(n)) * per_gpu
    achieved = flops / (avg_kernel_ms / 1e3) / 1e12
    peak = PEAK_F64_TFLOPS if args.dtype == "f64" else PEAK_F32_TFLOPS
    traffic, traffic_src = load_traffic(args.config, args.dtype)
    strat = model.resolve_strategy(per_gpu, args.dtype == "f64") if not fd else "aba_thread"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.scaling == "weak" else "strong", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic",
        "config": {"workload": f"{cfg['name']}: {'FD (ABA)' if fd else 'RNEA'} n={n} random serial chain, "
                               f"{per_gpu} states per GPU" if cfg['robot'] == 'random' and 'model' not in cfg else
                               f"{cfg['name']}: {cfg['robot']} n={n}, {per_gpu} states per GPU",
                   "n": n, "states_per_gpu": per_gpu, "global_batch": total, "gather_ms": gather_ms,
                   "parallelism": f"batch-sharded x{world} (no collective on the hot path)",
                   "strategy": strat, "robot_seed": 1000 + n if cfg["robot"] == "random" else cfg["robot"],
                   "state_seed": cfg["seed"], "l2": l2_note},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes": (32 if args.dtype == "f64" else 16) * n * per_gpu,
                     "flops_per_eval": lean_flops_fd(n) if fd else lean_flops_id(n),
                     "peak_basis": "148 SM x 64 DFMA/clk x 2 x 1.965 GHz (guide unit counts; measured DFMA "
                                   "microbench 34.0 TF/s, profiles/r01/peaks_alu.jsonl)"
                                   + ("; fp32 = 2x" if args.dtype == "f32" else ""),
                     "kernel_ms": avg_kernel_ms,
                     "algorithmic_hbm_gbs": 32 * n * per_gpu / (avg_kernel_ms / 1e3) / 1e9
                                            * (0.5 if args.dtype == "f32" else 1)},
        "clocks": clock.summary(),
        "gpu_launches": launches,
        "e2e": e2e,
    }
    if world > 1:
        pass                                        # the CPU baseline is an N = 1 figure (rank 0 only)
    elif not args.no_cpu_baseline and fd:
        line["cpu_baseline"] = cpu_baseline_fd(robot, g, cfg, n, args.cpu_seconds)
    elif not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(robot, g, cfg, n, args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
