"""Split one kernel's SASS (cuobjdump -sass) into basic blocks and print the
instruction mix of the large ones (loop bodies).  usage: sass_blocks.py file.sass func_substr [min]"""
import collections, re, sys

txt = open(sys.argv[1]).read().split("\n")
want, mn = sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 150
ins, on = [], False
for l in txt:
    if "Function :" in l:
        on = want in l
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if on and m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
targets = set()
for a, s in ins:
    m = re.search(r"BRA (?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", s)
    if m and m.group(1):
        targets.add(int(m.group(1), 16))
blocks, cur = [], []
for a, s in ins:
    if a in targets and cur:
        blocks.append(cur); cur = []
    cur.append((a, s))
    if "BRA" in s or "EXIT" in s:
        blocks.append(cur); cur = []
if cur:
    blocks.append(cur)
for b in blocks:
    if len(b) < mn:
        continue
    c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", s).split()[0].split(".")[0] for _, s in b)
    fp = c["DFMA"] + c["DMUL"] + c["DADD"]
    print(f"block {b[0][0]:#x}-{b[-1][0]:#x} n={len(b)} fp64={fp} (dfma {c['DFMA']} dmul {c['DMUL']} dadd {c['DADD']})",
          c.most_common(16))
