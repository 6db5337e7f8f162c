"""Multi-GPU slab decomposition of the particle path.

One process per GPU (torch.distributed; NCCL on B200s, gloo in the CPU tests).
Rank r owns the particles whose x-cell index lies in [b_r, b_{r+1}) — slabs of
whole cell planes, bounds balanced on the particle-count histogram — and keeps
GHOSTS: copies of the particles in the two cell planes beyond each face. Two
planes make the density of the first ghost plane complete, so one exchange per
step suffices for the two-pass WCSPH deck (density/EOS, then momentum, which
reads rho/p of neighbours up to one plane away). Per step:

  1. the physics step on owned + ghost particles (ghost results are discarded);
  2. MIGRATION: owned particles whose cell left the slab go to the neighbour;
  3. GHOSTS: owned particles in the first/last two planes go to the neighbours;
  4. reload the local set (owned + ghosts) keyed by global id, so cell lists keep
     ascending GLOBAL index order and every sum runs in the single-GPU order.

x is a ring when periodic (ghost positions stay true positions; the sweep's
periodic images do the rest), a line otherwise. The reference has no domain
decomposition; this is new.

The rank logic is written against a small backend interface so it runs both on
the CUDA library (GpuBackend, device rows as torch tensors, NCCL) and, in the
CPU tests, on the oracle (tests/slab_oracle.py, gloo).
"""
from __future__ import annotations

import math

import numpy as np


def balanced_bounds(cell_x: np.ndarray, ncx: int, world: int) -> list[int]:
    """Slab bounds [b_0=0, ..., b_world=ncx] of whole x-cell planes with ~equal counts."""
    return bounds_from_hist(np.bincount(cell_x, minlength=ncx), ncx, world)


def bounds_from_hist(hist: np.ndarray, ncx: int, world: int) -> list[int]:
    """balanced_bounds from a per-plane particle-count histogram (length ncx)."""
    cum = np.cumsum(np.asarray(hist, dtype=np.int64))
    total = cum[-1] if len(cum) else 0
    bounds = [0]
    for r in range(1, world):
        b = int(np.searchsorted(cum, total * r / world, side="left")) + 1
        b = max(b, bounds[-1] + 2)  # every slab at least two planes wide
        bounds.append(min(b, ncx - 2 * (world - r)))
    bounds.append(ncx)
    return bounds


def cell_x_of(x: np.ndarray, lo: float, cs: float, n: int, periodic: bool) -> np.ndarray:
    """particle_system.cpp:20-31 on the host (same IEEE division + floor)."""
    c = np.floor((x - lo) / cs).astype(np.int64)
    if periodic:
        return np.mod(c, n)
    return np.clip(c, 0, n - 1)


class Exchanger:
    """Variable-size row exchange with the left/right neighbours."""

    def __init__(self, dist, rank, world, periodic, device):
        self.dist, self.rank, self.world, self.periodic = dist, rank, world, periodic
        self.device = device
        self.left = (rank - 1) % world if (periodic or rank > 0) else None
        self.right = (rank + 1) % world if (periodic or rank < world - 1) else None

    def allreduce_sum(self, t):
        """Element-wise sum of a small int64 tensor over the ranks (in place)."""
        if self.world > 1:
            self.dist.all_reduce(t)
        return t

    def swap(self, to_left, to_right, width):
        """Send row blocks to the neighbours; return (from_left, from_right).

        Sends are posted [to_left, to_right] and receives [from_right, from_left]:
        P2P messages between one pair of ranks match in posting order, and on a
        2-rank ring the left and right neighbour are the same rank (my to_left is
        its from_right)."""
        import torch
        d = self.dist
        if self.world == 1:
            return None, None
        dev = self.device
        n_l = 0 if to_left is None else to_left.shape[0]
        n_r = 0 if to_right is None else to_right.shape[0]
        cnt_sl = torch.tensor([n_l], dtype=torch.int64, device=dev)
        cnt_sr = torch.tensor([n_r], dtype=torch.int64, device=dev)
        cnt_rl = torch.zeros(1, dtype=torch.int64, device=dev)
        cnt_rr = torch.zeros(1, dtype=torch.int64, device=dev)
        ops = []
        if self.left is not None:
            ops.append(d.P2POp(d.isend, cnt_sl, self.left))
        if self.right is not None:
            ops.append(d.P2POp(d.isend, cnt_sr, self.right))
            ops.append(d.P2POp(d.irecv, cnt_rr, self.right))
        if self.left is not None:
            ops.append(d.P2POp(d.irecv, cnt_rl, self.left))
        for w in d.batch_isend_irecv(ops):
            w.wait()
        from_left = torch.empty((int(cnt_rl.item()), width), dtype=torch.float64, device=dev)
        from_right = torch.empty((int(cnt_rr.item()), width), dtype=torch.float64, device=dev)
        ops = []
        if self.left is not None and n_l:
            ops.append(d.P2POp(d.isend, to_left.contiguous(), self.left))
        if self.right is not None and n_r:
            ops.append(d.P2POp(d.isend, to_right.contiguous(), self.right))
        if self.right is not None and from_right.shape[0]:
            ops.append(d.P2POp(d.irecv, from_right, self.right))
        if self.left is not None and from_left.shape[0]:
            ops.append(d.P2POp(d.irecv, from_left, self.left))
        if ops:
            for w in d.batch_isend_irecv(ops):
                w.wait()
        return (from_left if self.left is not None else None,
                from_right if self.right is not None else None)


class SlabRank:
    """The per-rank driver. `backend` provides:
        width, col_gid, col_ghost          row layout
        load(rows)                         replace the local particle set (rows keyed by gid)
        select(c_lo, c_hi, ghost)          rows of active particles with x-cell in [c_lo, c_hi)
                                           (taken mod ncx when periodic) and ghost flag == ghost
        step()                             one physics step on the local set
        cat(blocks)                        row concatenation (None entries skipped)
    """

    GHOST_PLANES = 2

    def __init__(self, backend, exchanger, bounds, ncx, periodic, rebalance_every=0,
                 x_lo=0.0, cell_size=None):
        """rebalance_every > 0 (needs x_lo, cell_size: the x origin and size of the cell
        planes) re-balances the slab bounds on the global x-plane histogram every that many
        steps (the dam-break fluid moves right)."""
        self.b = backend
        self.x = exchanger
        self.r = exchanger.rank
        self.bounds = list(bounds)
        self.lo_c, self.hi_c = bounds[self.r], bounds[self.r + 1]
        self.ncx, self.periodic = ncx, periodic
        self.rebalance_every = rebalance_every
        if rebalance_every and cell_size is None:
            raise ValueError("rebalancing needs the x cell-plane geometry (x_lo, cell_size)")
        self.x_lo, self.cs = x_lo, cell_size
        self.steps = 0
        self.rebalances = 0  # bound changes so far

    def _sel(self, c0, c1, ghost):
        """Rows with x-cell in [c0, c1) (wrapping on a ring)."""
        if not self.periodic:
            c0, c1 = max(c0, 0), min(c1, self.ncx)
            return self.b.select(c0, c1, ghost) if c1 > c0 else None
        n = self.ncx
        if c1 <= c0:
            return None
        if c1 - c0 >= n:
            return self.b.select(0, n, ghost)
        # shift the range so that 0 <= c0 < n, then split it at the seam
        k = c0 // n
        c0, c1 = c0 - k * n, c1 - k * n
        parts = [self.b.select(c0, min(c1, n), ghost)]
        if c1 > n:
            parts.append(self.b.select(0, c1 - n, ghost))
        return self.b.cat(parts)

    def exchange(self):
        """Migration + ghost refresh after a step (steps 2-4 of the module doc)."""
        g = self.GHOST_PLANES
        keep = self.b.select(self.lo_c, self.hi_c, 0)
        # particles move less than a cell per step (CFL); look one ghost width out
        to_left = self._sel(self.lo_c - g, self.lo_c, 0)
        to_right = self._sel(self.hi_c, self.hi_c + g, 0)
        if self.x.world == 1 and self.periodic:
            to_left = to_right = None  # one rank owns every plane
        from_left, from_right = self.x.swap(to_left, to_right, self.b.width)
        owned = self.b.cat([keep, from_left, from_right])
        self.b.load(owned)
        if self.rebalance_every and self.x.world > 1 and self.steps % self.rebalance_every == 0:
            owned = self.rebalance(owned)
        gl = self._sel(self.lo_c, self.lo_c + g, 0)
        gr = self._sel(self.hi_c - g, self.hi_c, 0)
        if self.x.world == 1:
            self.b.load(owned)
            return
        from_left, from_right = self.x.swap(gl, gr, self.b.width)
        ghosts = [self.b.mark_ghost(blk) for blk in (from_left, from_right) if blk is not None]
        self.b.load(self.b.cat([owned] + ghosts))

    def plane_hist(self, rows):
        """Global per-x-plane count of owned particles (cell_x_of on the rows' x column)."""
        import torch
        x = rows[:, 0]
        c = torch.floor((x - self.x_lo) / self.cs).to(torch.int64)
        c = torch.remainder(c, self.ncx) if self.periodic else c.clamp(0, self.ncx - 1)
        h = torch.bincount(c, minlength=self.ncx)
        return self.x.allreduce_sum(h.to(torch.int64)).cpu().numpy()

    def rebalance(self, owned):
        """New bounds from the global plane histogram; owned particles then hop rank by rank
        toward their new owner (a bound may move past a whole neighbouring slab). The local
        set holds owned particles only (ghosts are refreshed by the caller); every particle
        keeps its global id, so sums stay in the single-GPU order."""
        import torch
        hist = self.plane_hist(owned)
        new = bounds_from_hist(hist, self.ncx, self.x.world)
        if new == self.bounds:
            return owned
        total = int(hist.sum())
        self.bounds = new
        self.lo_c, self.hi_c = new[self.r], new[self.r + 1]
        self.rebalances += 1
        lo, hi, n = self.lo_c, self.hi_c, self.ncx
        if self.periodic:
            out = n - (hi - lo)          # planes outside the slab, hi .. lo-1 around the ring
            right = (out + 1) // 2       # the nearer half goes right, the rest left
            rng_r, rng_l = (hi, hi + right), (hi + right, hi + out)
        else:
            rng_r, rng_l = (hi, n), (0, lo)
        for _ in range(self.x.world + 1):
            to_right = self._sel(*rng_r, 0)
            to_left = self._sel(*rng_l, 0)
            cnt = sum(0 if t is None else int(t.shape[0]) for t in (to_left, to_right))
            pending = self.x.allreduce_sum(torch.tensor([cnt], dtype=torch.int64,
                                                        device=self.x.device))
            if int(pending.item()) == 0:
                got = self.x.allreduce_sum(torch.tensor([int(owned.shape[0])], dtype=torch.int64,
                                                        device=self.x.device))
                if int(got.item()) != total:  # a particle duplicated or dropped in transit
                    raise RuntimeError(f"slab rebalance: {int(got.item())} owned rows after the "
                                       f"hops, {total} before")
                return owned
            keep = self.b.select(lo, hi, 0)
            from_left, from_right = self.x.swap(to_left, to_right, self.b.width)
            owned = self.b.cat([keep, from_left, from_right])
            self.b.load(owned)
        raise RuntimeError("slab rebalance: particles still misplaced after world+1 hops")

    def step(self):
        self.b.step()
        self.steps += 1
        self.exchange()


def initial_rows(scene, field_names, bounds, rank, ncx, periodic, ghost_planes=2):
    """Host rows (owned + ghosts) of `rank` from the full scene; columns: r, fields..., gid, ghost."""
    n = scene.n
    lo, cs = scene.min_cells[0] * scene.cell_size[0], scene.cell_size[0]
    cx = cell_x_of(scene.pos[0], lo, cs, ncx, periodic)
    b0, b1 = bounds[rank], bounds[rank + 1]
    owned = (cx >= b0) & (cx < b1)
    if periodic:
        dl = np.mod(b0 - cx, ncx)  # planes to the left of the slab
        dr = np.mod(cx - b1, ncx)
        ghost = ~owned & (((dl >= 1) & (dl <= ghost_planes)) | (dr < ghost_planes))
    else:
        ghost = ~owned & (((cx >= b0 - ghost_planes) & (cx < b0)) |
                          ((cx >= b1) & (cx < b1 + ghost_planes)))
    cols = [scene.pos]
    for name in field_names:
        cols.append(np.asarray(scene.fields[name], dtype=np.float64).reshape(-1, n))
    cols.append(np.arange(n, dtype=np.float64)[None, :])            # gid
    cols.append(np.where(ghost, 1.0, 0.0)[None, :])                  # ghost flag
    rows = np.concatenate(cols, axis=0).T
    sel = owned | ghost
    if len(bounds) == 2:  # single rank: no ghosts at all
        sel = owned
        rows[:, -1] = 0.0
    return np.ascontiguousarray(rows[sel])


class GpuBackend:
    """Backend over the CUDA library; rows are device tensors (torch, float64)."""

    def __init__(self, ctx, wcsph_params, field_names, gid_name="gid", ghost_name="ghost"):
        import torch
        self.torch = torch
        self.ctx = ctx
        self.p = wcsph_params
        self.gid = ctx.fields[gid_name].id
        self.ghost_id = ctx.fields[ghost_name].id
        self.width = ctx.L.nau_row_width(ctx.h)
        self.col_gid = self.width - 2
        self.col_ghost = self.width - 1
        self.device = f"cuda:{torch.cuda.current_device()}"

    def load(self, rows):
        rows = rows.contiguous()
        self.ctx._check(self.ctx.L.nau_load_rows(self.ctx.h, rows.data_ptr(), rows.shape[0],
                                                 self.gid))
        self.ctx.n = rows.shape[0]
        self._rows_keepalive = rows

    def select(self, c0, c1, ghost):
        import ctypes as C
        torch = self.torch
        slots = torch.empty(max(1, self.ctx.n), dtype=torch.int32, device=self.device)
        cnt = C.c_long(0)
        self.ctx._check(self.ctx.L.nau_select(self.ctx.h, 0, float(c0), float(c1), self.ghost_id,
                                              float(ghost), float(ghost), slots.data_ptr(),
                                              C.byref(cnt)))
        m = cnt.value
        rows = torch.empty((m, self.width), dtype=torch.float64, device=self.device)
        if m:
            self.ctx._check(self.ctx.L.nau_pack_rows(self.ctx.h, slots.data_ptr(), m,
                                                     rows.data_ptr()))
        return rows

    def mark_ghost(self, rows):
        rows = rows.clone()
        rows[:, self.col_ghost] = 1.0
        return rows

    def cat(self, blocks):
        blocks = [b for b in blocks if b is not None and b.shape[0]]
        if not blocks:
            return self.torch.empty((0, self.width), dtype=self.torch.float64, device=self.device)
        return self.torch.cat(blocks, 0)

    def step(self):
        if callable(self.p):
            self.p()  # a deck step callback (e.g. the DEM deck)
        else:
            self.ctx.wcsph_step(self.p)
