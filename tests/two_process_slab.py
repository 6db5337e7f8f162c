"""Worker of tests/test_gpu_two_process.py: one slab rank per PROCESS, all on GPU 0, rows
exchanged over gloo (host-staged; no kernel of one rank waits on another's). Runs the
bench's DamBreakSlab driver — the real Exchanger, GpuBackend and stream handling — and
rank 0 compares the gathered owned particles with a single-context run, bitwise."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1710_08259_b200 import nau, scenes  # noqa: E402

STEPS = 7


def scene():
    sc = scenes.dam_break(2, dx=0.05, fluid=(1.0, 1.0), tank=(2.0, 1.6))
    sc.fields["v"][0, : sc.params["n_fluid"]] = 6.0  # fluid crosses the slab faces
    return sc


def nbody(d, fast):
    """cfg4's sharded path: broadcast-pipelined source chunks (slab.pipelined_sources +
    nau_gravity_sources_part) against the plain leapfrog, bitwise."""
    n = 1536  # divisible by 2 and 3
    ctx = nau.Context(0)
    ctx.set_mode(fast)
    sh = bench.GravityShard(d)
    sh.sc = scenes.plummer(n=n)
    sh.setup(ctx)
    for _ in range(3):
        sh.step(ctx)
    ctx.sync()
    mine = np.concatenate([ctx.download("r"), ctx.download("v"), ctx.download("a")]).T.copy()
    parts = [None] * d.world
    dist.gather_object(mine, parts if d.rank == 0 else None, dst=0)
    ok = True
    if d.rank == 0:
        plain = bench.Gravity()
        plain.sc = scenes.plummer(n=n)
        c1 = nau.Context(0)
        c1.set_mode(fast)
        plain.setup(c1)
        for _ in range(3):
            plain.step(c1)
        ref = np.concatenate([c1.download("r"), c1.download("v"), c1.download("a")]).T
        ok = np.array_equal(np.concatenate(parts), ref)
        print("two_process_slab", "OK" if ok else "MISMATCH", d.world, "ranks nbody",
              "fast" if fast else "exact", flush=True)
    return ok


def main():
    fast = sys.argv[1] == "fast"
    os.environ["NAU_BENCH_DEVICE"] = "0"
    os.environ["NAU_DIST_BACKEND"] = "gloo"
    d = bench.Dist()
    if len(sys.argv) > 2 and sys.argv[2] == "nbody":
        ok = nbody(d, fast)
        d.close()
        sys.exit(0 if ok else 1)
    ctx = nau.Context(0)
    ctx.set_mode(fast)
    sl = bench.DamBreakSlab(2, d)
    sl.sc = scene()
    sl.REBALANCE_EVERY = 3
    sl.setup(ctx)
    for _ in range(STEPS):  # default stream current, as in the bench's warm-up steps
        sl.step(ctx)
    ctx.sync()
    own = ctx.download("ghost")[0] == 0
    mine = np.concatenate([ctx.download("gid")[:, own], ctx.download("r")[:, own],
                           ctx.download("v")[:, own]]).T.copy()
    parts = [None] * d.world
    dist.gather_object(mine, parts if d.rank == 0 else None, dst=0)
    ok = True
    if d.rank == 0:
        plain = bench.DamBreak(2)
        plain.sc = scene()
        c1 = nau.Context(0)
        c1.set_mode(fast)
        plain.setup(c1)
        for _ in range(STEPS):
            plain.step(c1)
        ref = np.concatenate([c1.download("r"), c1.download("v")]).T
        allp = np.concatenate(parts)
        gid = allp[:, 0].astype(int)
        ok = np.array_equal(np.sort(gid), np.arange(ref.shape[0])) and np.array_equal(allp[:, 1:], ref[gid])
        print("two_process_slab", "OK" if ok else "MISMATCH", d.world, "ranks", "fast" if fast else "exact",
              "rebalances", sl.rank_drv.rebalances, flush=True)
    d.close()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
