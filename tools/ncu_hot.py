"""Hottest SASS instructions of one kernel from an ncu report's source page.

    ncu -i rep.ncu-rep --page source --csv --print-source sass -k regex:NAME > src.csv
    python tools/ncu_hot.py src.csv [top]
Prints per-instruction stall samples (top N) and the kernel's stall-reason totals.
"""
import csv
import sys
from collections import Counter


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    cols = rows[hdr]
    ix = {c: i for i, c in enumerate(cols)}
    stall_cols = [c for c in cols if c.startswith("stall_") and "Not Issued" not in c]
    tot = Counter()
    recs = []
    for n, r in enumerate(rows[hdr + 1:]):
        if len(r) < len(cols) or r[0] == "Address":
            continue
        s = int(r[ix["# Samples"]] or 0)
        st = {c: int(r[ix[c]] or 0) for c in stall_cols}
        for c, v in st.items():
            tot[c] += v
        recs.append((s, n, r[ix["Source"]].strip(), st, int(r[ix["Instructions Executed"]] or 0)))
    allsamp = sum(s for s, *_ in recs)
    print("samples", allsamp)
    print("stall totals:", ", ".join(f"{c[6:]} {v * 100 // max(allsamp, 1)}%" for c, v in tot.most_common(8)))
    for s, n, src, st, ie in sorted(recs, reverse=True)[:top]:
        why = ", ".join(f"{c[6:]} {v}" for c, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
        print(f"{s:7d} {s * 100 / allsamp:5.1f}%  #{n:4d} x{ie:9d}  {src[:60]:60s} {why}")


if __name__ == "__main__":
    main()
