"""Map the top stall-sampled SASS instructions of an ncu source page (sass, csv)
to CUDA source lines via the cubin's line table (nvdisasm -g).

usage: sass_lines.py SOURCE.csv OBJ.o FUNC_SUBSTR [top]
"""
import csv
import os
import re
import subprocess
import sys
import tempfile

src_csv, obj, func = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
rows = list(csv.reader(open(src_csv)))
hdr, data = rows[1], rows[2:]
iss = hdr.index("Warp Stall Sampling (All Samples)")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][0], 16)
tot = sum(float(r[iss] or 0) for r in data)

d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
line_of, cur_line, on = {}, "?", False
for l in dis.split("\n"):
    if l.startswith("//---------------------"):
        on = func in l
        continue
    if not on:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        line_of[int(m.group(1), 16)] = cur_line
agg = {}
for r in data:
    v = float(r[iss] or 0)
    if v <= 0:
        continue
    ln = line_of.get(int(r[0], 16) - base, "?")
    a = agg.setdefault(ln, [0.0, {}])
    a[0] += v
    for h in cols:
        a[1][h] = a[1].get(h, 0) + float(r[hdr.index(h)] or 0)
print(f"stall samples by source line (of {tot:.0f}):")
for ln, (v, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    worst = sorted(st.items(), key=lambda x: -x[1])[:2]
    print(f"  {100 * v / tot:5.1f}%  {ln:24s} " + "  ".join(f"{k[6:]} {100 * x / tot:.1f}" for k, x in worst))
