"""Executed FP64 flops of one kernel from an ncu --set full report (FMA = 2):
the per-cycle SASS DFMA / DMUL / DADD rates (summed over SMSPs) x elapsed
cycles.  (The fp32 op counters do not include the packed FFMA2 / FMUL2, so the
tool reports FP64 only.)  usage: ncu_flops.py REPORT.ncu-rep UNITS LINKS
(units = states per launch)."""
import csv
import subprocess
import sys

rep, units, links = sys.argv[1], float(sys.argv[2]), float(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, unit, val = rows[0], rows[1], rows[2]
m = {h: val[i] for i, h in enumerate(hdr)}
u = {h: unit[i] for i, h in enumerate(hdr)}


def f(name):
    return float(m[name].replace(",", ""))


cyc = f("smsp__cycles_elapsed.avg")                 # per-SMSP elapsed cycles
res = {}
for p, (fma, mul, add) in {"fp64": ("dfma", "dmul", "dadd")}.items():
    rate = lambda op: f(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")  # noqa: E731
    n_fma, n_mul, n_add = (rate(o) * cyc for o in (fma, mul, add))
    res[p] = (2 * n_fma + n_mul + n_add, n_fma + n_mul + n_add)
scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
dur = f("gpu__time_duration.sum") * scale.get(u.get("gpu__time_duration.sum", "ns"), 1e-9)
for p, (flops, inst) in res.items():
    if flops == 0:
        continue
    print(f"{p}: executed {flops / units:.0f} flops/unit ({flops / units / links:.1f} per link), "
          f"{inst / units / links:.1f} instructions per link"
          + (f", {flops / dur / 1e12:.2f} TFLOP/s over the ncu duration" if dur else ""))
