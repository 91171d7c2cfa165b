"""Write profiles/ncu_traffic.json from ncu summaries (tools/ncu_summary.py output):
dram__bytes_read.sum + dram__bytes_write.sum of the captured launch, per bench
config.  usage: ncu_traffic.py KEY=SUMMARY.txt [KEY=SUMMARY.txt ...]"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {"_doc": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from one "
               "ncu --set full capture (--clock-control none, tools/run_ncu_one.sh); bench.py copies the "
               "matching entry into roofline.traffic and its source into roofline.traffic_source"}
for arg in sys.argv[1:]:
    key, path = arg.split("=", 1)
    tot = 0.0
    for line in open(path):
        m = re.match(r"\s*dram__bytes_(read|write)\.sum\s+([\d.]+)\s+(\w+)", line)
        if m:
            tot += float(m.group(2)) * UNIT[m.group(3)]
    out[key] = int(round(tot))
    out[key + "_source"] = os.path.relpath(path, ROOT)
with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
