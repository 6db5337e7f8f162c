"""Shape of the neighbour lists a bench workload builds (nau_list_stats).

    python tools/list_probe.py --config 2
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1710_08259_b200 import nau  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    wl = bench.make_workload(args.config)
    ctx = nau.Context(0)
    ctx.set_mode(True)
    wl.setup(ctx)
    for _ in range(args.steps):
        wl.step(ctx)
    ctx.sync()
    st = ctx.list_stats()
    st["path"] = ctx.wcsph_path
    print(json.dumps(st))


if __name__ == "__main__":
    main()
