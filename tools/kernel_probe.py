"""Per-kernel times of the cfg2 density / momentum passes for timing-only library
variants whose results are wrong on purpose (device errors are caught and ignored:
the pair bodies are branch-free, so the work does not depend on the values).

    NAU_LIB=build/var/<name>/libnau_b200.so python tools/kernel_probe.py [--config 2]
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
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    wl = bench.make_workload(args.config)
    ctx = nau.Context(0)
    ctx.set_mode(True)
    wl.setup(ctx)

    def quiet(fn):
        try:
            fn()
        except nau.NauError:
            pass

    quiet(lambda: (ctx.wcsph_pass(wl.p, 0), ctx.wcsph_pass(wl.p, 1), ctx.sync()))
    ctx.profile(True)
    for _ in range(args.reps):  # positions never move: no integrator pass
        quiet(lambda: (ctx.wcsph_pass(wl.p, 0), ctx.wcsph_pass(wl.p, 1), ctx.sync()))
    out = {}
    for cls, name in ((200, "density"), (201, "momentum"), (302, "list build")):
        ms, cnt = ctx.profile_ms(cls)
        out[name] = round(ms / max(cnt, 1), 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
