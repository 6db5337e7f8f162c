"""Can the list build + density pass of one slot range share the SMs with the momentum
pass of another? Two contexts (two copies of cfg2, one stream each): A repeats
cells + list + density, B repeats the momentum pass; sequential vs interleaved issue.

    python tools/overlap_probe.py [--dx 0.005]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1710_08259_b200 import nau  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=6)
    args = ap.parse_args()
    A, B = nau.Context(0), nau.Context(0)
    wa, wb = bench.make_workload(2), bench.make_workload(2)
    for c, w in ((A, wa), (B, wb)):
        c.set_mode(True)
        w.setup(c)
        c.wcsph_pass(w.p, 0)
        c.wcsph_pass(w.p, 1)
        c.sync()

    def passA():
        A.boundary_shift()     # marks the cells dirty: pass 0 rebuilds cells + list
        A.wcsph_pass(wa.p, 0)

    def timed(fn):
        A.sync(); B.sync()
        t0 = time.perf_counter()
        fn()
        A.sync(); B.sync()
        return (time.perf_counter() - t0) * 1e3 / args.reps

    def seqA():
        for _ in range(args.reps):
            passA()

    def seqB():
        for _ in range(args.reps):
            B.wcsph_pass(wb.p, 1)

    def both():
        for _ in range(args.reps):
            passA()
            B.wcsph_pass(wb.p, 1)

    timed(both)
    out = {"A cells+list+density": round(timed(seqA), 3), "B momentum": round(timed(seqB), 3),
           "interleaved": round(timed(both), 3)}
    out["sum"] = round(out["A cells+list+density"] + out["B momentum"], 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
