"""Run a few steps of a bench workload (for ncu launch lists / captures).

    python tools/profile_step.py --config 2 --steps 2 [--mode fast|exact]
Exits 0 only if the steps ran cleanly (device errors surface at sync).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1710_08259_b200 import nau  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--mode", default="fast", choices=["fast", "exact"])
    args = ap.parse_args()
    wl = bench.make_workload(args.config)
    ctx = nau.Context(0)
    ctx.set_mode(args.mode == "fast")
    wl.setup(ctx)
    for _ in range(args.steps):
        wl.step(ctx)
    ctx.sync()
    print("ok", args.config, args.mode, args.steps, "launches", ctx.launches)


if __name__ == "__main__":
    main()
