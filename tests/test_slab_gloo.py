"""CPU tests of the multi-GPU slab decomposition (paper_1710_08259_b200/slab.py):
world_size 2 over gloo, each rank stepping its slab (+ ghosts) with the oracle
backend. After several steps with particles crossing slab faces, the owned
particles gathered by global id must equal a single-rank run BITWISE — the slab
path keeps every sum in the single-GPU (reference) order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import slab_oracle
from paper_1710_08259_b200 import scenes, slab

STEPS = 12


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make_scene(kind):
    if kind == "dam":
        sc = scenes.dam_break(2, dx=0.05, fluid=(1.0, 1.0), tank=(2.0, 1.6))
        sc.fields["v"][0, : sc.params["n_fluid"]] = 6.0  # push fluid across slab faces
        sc.params["dt"] = 5e-4
        return sc, False
    # periodic x: a fluid layer over a 3-layer floor, sheared fast x-velocity so
    # particles wrap around the ring and cross both slab faces
    # "ring30": the same layer on a 30-plane ring (re-balanced planes cross the seam)
    planes = 30 if kind == "ring30" else 10
    base = scenes.dam_break(2, dx=0.05, fluid=(2.0, 0.5), tank=(2.0, 1.0))
    dx = 0.05
    nx = 4 * planes
    fx, fy = np.meshgrid((np.arange(nx) + 0.5) * dx, (np.arange(10) + 0.5) * dx, indexing="xy")
    wx, wy = np.meshgrid((np.arange(nx) + 0.5) * dx, -(np.arange(3) + 0.5) * dx, indexing="xy")
    pos = np.stack([np.concatenate([fx.ravel(), wx.ravel()]), np.concatenate([fy.ravel(), wy.ravel()])])
    n, nf = pos.shape[1], fx.size
    mask = np.zeros(n)
    mask[:nf] = 1.0
    v = np.zeros((2, n))
    v[0, :nf] = 2.0 + pos[1, :nf]
    sc = scenes.Scene("periodic_layer", 2, [0, -1], [planes, 6], [0.2, 0.2], [0, 2], pos,
                      fields={"rho": np.full(n, 1000.0), "p": np.zeros(n), "v": v,
                              "vdot": np.zeros((2, n)), "mask": mask},
                      params=dict(base.params, dt=5e-4))
    return sc, True


def run_rank(rank, world, port_, kind, out, rebalance=0, skew=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    sc, periodic = make_scene(kind)
    ncx = sc.max_cells[0] - sc.min_cells[0]
    lo, cs = sc.min_cells[0] * sc.cell_size[0], sc.cell_size[0]
    cx = slab.cell_x_of(sc.pos[0], lo, cs, ncx, periodic)
    bounds = slab.balanced_bounds(cx, ncx, world)
    if skew:  # badly balanced start: every slab but the last two planes wide
        bounds = [2 * i for i in range(world)] + [ncx]
    be = slab_oracle.OracleBackend(sc, ncx, periodic)
    ex = slab.Exchanger(dist if world > 1 else None, rank, world, periodic, "cpu")
    r = slab.SlabRank(be, ex, bounds, ncx, periodic, rebalance_every=rebalance, x_lo=lo,
                      cell_size=cs)
    be.load(torch.from_numpy(slab.initial_rows(sc, slab_oracle.FIELDS, bounds, rank, ncx, periodic)))
    for _ in range(STEPS):
        r.step()
    owned = be.rows[(be.rows[:, be.col_ghost] == 0) & be.active]
    first = set(slab.initial_rows(sc, slab_oracle.FIELDS, bounds, rank, ncx, periodic)[:, -2].tolist())
    out[rank] = (owned, len(set(owned[:, -2].tolist()) ^ first), r.rebalances, r.bounds)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _worker(rank, world, port_, kind, q, rebalance, skew):
    out = {}
    run_rank(rank, world, port_, kind, out, rebalance, skew)
    q.put((rank, out[rank]))


def run_world(world, kind, rebalance=0, skew=False, info=None):
    if world == 1:
        out = {}
        run_rank(0, 1, 0, kind, out)
        return out[0][0], 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_, kind, q, rebalance, skew))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    moved = sum(res[r][1] for r in range(world))
    if info is not None:
        info.extend(res[r][2:] for r in range(world))
    return np.concatenate([res[r][0] for r in range(world)], axis=0), moved


@pytest.mark.parametrize("kind", ["dam", "periodic"])
def test_two_slabs_match_one_rank_bitwise(kind):
    one, _ = run_world(1, kind)
    two, moved = run_world(2, kind)
    assert moved > 0, "no particle changed slab: the test would not exercise migration"
    gid = one.shape[1] - 2
    one = one[np.argsort(one[:, gid])]
    two = two[np.argsort(two[:, gid])]
    assert len(np.unique(two[:, gid])) == len(two), "a particle is owned twice"
    np.testing.assert_array_equal(two[:, gid], one[:, gid])  # no particle lost
    np.testing.assert_array_equal(two, one)


@pytest.mark.parametrize("kind,world", [("dam", 3), ("periodic", 3), ("ring30", 3)])
def test_rebalanced_slabs_match_one_rank_bitwise(kind, world):
    """SURVEY.md §8(e) re-balancing: start from skewed bounds (two-plane slabs and one
    huge one), re-balance every 4 steps on the global plane histogram; bounds move by
    more than a whole slab, so particles hop over a rank, and results stay bitwise."""
    one, _ = run_world(1, kind)
    info = []
    many, _ = run_world(world, kind, rebalance=4, skew=True, info=info)
    assert all(n >= 1 for n, _ in info), "bounds never changed"
    assert len({tuple(b) for _, b in info}) == 1, "ranks disagree on the bounds"
    final = info[0][1]
    assert final != [0, 2, 4, final[-1]] and all(final[i + 1] - final[i] >= 2 for i in range(world))
    gid = one.shape[1] - 2
    one = one[np.argsort(one[:, gid])]
    many = many[np.argsort(many[:, gid])]
    assert len(np.unique(many[:, gid])) == len(many), "a particle is owned twice"
    np.testing.assert_array_equal(many, one)


def test_bounds_from_hist():
    h = np.array([0, 0, 5, 50, 50, 50, 50, 5, 0, 0])
    cx = np.repeat(np.arange(10), h)
    assert slab.bounds_from_hist(h, 10, 3) == slab.balanced_bounds(cx, 10, 3)


def test_balanced_bounds():
    cx = np.repeat(np.arange(10), [0, 0, 5, 50, 50, 50, 50, 5, 0, 0])
    b = slab.balanced_bounds(cx, 10, 2)
    assert b[0] == 0 and b[-1] == 10 and 3 <= b[1] <= 6
    b4 = slab.balanced_bounds(cx, 10, 4)
    assert all(b4[i + 1] - b4[i] >= 2 for i in range(4))
