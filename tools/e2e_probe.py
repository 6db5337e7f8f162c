"""Where the e2e leg of bench.py loses time: the cfg2 step timed through
timed_pipelined with (a) no copies, (b) uploads only, (c) downloads only, (d) both,
plus the per-kernel profile under (d). One JSON line per variant.

python tools/e2e_probe.py [--config 2] [--steps 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    from paper_1710_08259_b200 import nau

    dist = bench.Dist()
    wl = bench.make_workload(args.config, dist, False, False)
    ctx = nau.Context(0)
    ctx.set_mode(True)
    wl.setup(ctx)
    for _ in range(3):
        wl.e2e_step(ctx)
    ctx.sync()

    def up_only(c):
        c.upload_async("r", wl.h_r.data_ptr())
        c.upload_async("v", wl.h_v.data_ptr())
        wl.step(c)

    def down_only(c):
        wl.step(c)
        for k, t in wl.h_out.items():
            c.download_async(k, t.data_ptr())

    variants = {"step": wl.step, "up": up_only, "down": down_only, "e2e": wl.e2e_step}
    for name, fn in variants.items():
        ms = bench.timed_pipelined(ctx, fn, args.steps) / args.steps
        print(json.dumps({"variant": name, "ms_per_step": round(ms, 3)}), flush=True)
    # D2H bandwidth alone and under the step: one 379 MB copy on a side stream per step
    import torch
    nb = wl.d2h // 8
    dsrc = torch.empty(nb, dtype=torch.float64, device="cuda")
    hdst = torch.empty(nb, dtype=torch.float64).pin_memory()
    side = torch.cuda.Stream()
    main = torch.cuda.ExternalStream(ctx.L.nau_get_stream(ctx.h))
    for label, with_step in (("d2h alone", False), ("d2h under step", True)):
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ctx.sync()
        with torch.cuda.stream(main):
            s0.record(main)
        side.wait_event(s0)
        with torch.cuda.stream(side):
            c0.record(side)
            hdst.copy_(dsrc, non_blocking=True)
            c1.record(side)
        if with_step:
            wl.step(ctx)
        with torch.cuda.stream(main):
            s1.record(main)
        torch.cuda.synchronize()
        ctx.sync()
        print(json.dumps({"variant": label, "copy_ms": round(c0.elapsed_time(c1), 3),
                          "GBps": round(wl.d2h / c0.elapsed_time(c1) / 1e6, 1),
                          "step_ms": round(s0.elapsed_time(s1), 3)}), flush=True)
    ctx.profile(True)
    bench.timed_pipelined(ctx, wl.e2e_step, args.steps)
    prof = {wl.kernels[c][0]: [round(x, 3) for x in ctx.profile_ms(c)] for c in wl.kernels}
    ctx.profile(False)
    print(json.dumps({"variant": "e2e kernels (total ms, launches)", "kernels": prof}))


if __name__ == "__main__":
    main()
