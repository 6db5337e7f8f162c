"""Dynamic opcode mix of one kernel from an ncu source page (instructions executed per
opcode, and the top lines by executed count / stall samples).

    ncu -i rep.ncu-rep --page source --csv --print-source sass --launch-skip K --launch-count 1 > src.csv
    python tools/ncu_mix.py src.csv
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
cols = rows[hdr]
ix = {c: i for i, c in enumerate(cols)}
recs, seen = [], set()
for r in rows[hdr + 1:]:
    if len(r) < len(cols) or r[0] == "Address" or r[0] in seen:
        continue
    seen.add(r[0])
    recs.append((int(r[ix["Instructions Executed"]] or 0), r[ix["Source"]].strip(), int(r[ix["# Samples"]] or 0)))
tot = sum(x[0] for x in recs)
samp = sum(x[2] for x in recs)
print("warp instructions", tot, "samples", samp)
c = Counter()
for n, src, _ in recs:
    t = src.split()
    op = t[1] if t and t[0].startswith("@") else (t[0] if t else "")
    c[op.split(".")[0]] += n
print(" ".join(f"{k}:{v / tot * 100:.1f}%" for k, v in c.most_common(22)))
print("top by samples:")
for n, src, s in sorted(recs, key=lambda x: -x[2])[:14]:
    print(f"  {s / samp * 100:5.1f}%  x{n:9d}  {src[:70]}")
