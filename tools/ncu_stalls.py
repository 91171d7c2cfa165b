"""Summarise ncu --page source --csv: stall reasons in total and the top instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {h: hdr.index(h) for h in cols}
tot = {h: sum(float(r[idx[h]] or 0) for r in data) for h in cols}
S = sum(tot.values())
print("stall totals (% of samples):")
for h, v in sorted(tot.items(), key=lambda x: -x[1]):
    if v > 0:
        print(f"  {h:28s} {100 * v / S:6.2f}")
isrc, iss = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
print("top instructions:")
for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:top]:
    worst = max(cols, key=lambda h: float(r[idx[h]] or 0))
    print(f"  {float(r[iss]) / S * 100:5.2f}%  {r[0]}  {r[isrc][:60]:60s} {worst}")
