"""Split an ncu source-page CSV (SASS) into address ranges and print per-range instruction counts
and stall samples (development aid for warp-specialised kernels).
usage: ncu_roles.py file.source.csv [split_addr_hex ...]"""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
iA, iS, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
cuts = [int(x, 16) for x in sys.argv[2:]]
base = int(data[0][iA], 16)
def rng(a):
    off = a - base
    return sum(1 for c in cuts if off >= c)
agg = collections.defaultdict(lambda: collections.Counter())
for r in data:
    try: a = int(r[iA], 16); e = int(r[iE])
    except ValueError: continue
    g = rng(a)
    agg[g]["inst"] += e
    s = re.sub(r'^@!?U?P\w+\s+', '', r[iS].strip())
    if re.match(r'D(FMA|MUL|ADD)', s): agg[g]["fp64"] += e
    for h in st:
        try: agg[g][h] += int(r[hdr.index(h)] or 0)
        except ValueError: pass
for g in sorted(agg):
    c = agg[g]; tot = sum(c[h] for h in st) or 1
    top = sorted(((c[h] / tot * 100, h[6:]) for h in st), reverse=True)[:7]
    print(f"range {g}: inst {c['inst']/1e6:.1f}M fp64 {c['fp64']/1e6:.1f}M samples {tot}  " +
          " ".join(f"{n} {p:.0f}%" for p, n in top))
