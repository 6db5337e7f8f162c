"""Multi-GPU slab decomposition of the particle path.

One process per GPU (torch.distributed; NCCL on B200s, gloo in the CPU tests).
Rank r OWNS the particles whose x lies in [X_r, X_{r+1}) — x-threshold slabs,
bounds balanced on a fine x-histogram of particle counts — and holds GHOSTS:
copies of its neighbours' particles within one interaction radius R of its faces
(flag 1: owned by the left neighbour, flag 2: by the right one). Ghosts take part
in every neighbour sum but are never evaluated or integrated (nau_set_ghost_field).
Per WCSPH step (the §8(e) schedule):

  1. density/EOS pass on the owned particles (ghosts are neighbours);
  2. HALO VALUES: each owner sends (rho, p) of its particles within R of a face to
     that neighbour, which writes them into its ghosts (nau_wcsph_ghost_update);
  3. momentum pass, symplectic update (owned only);
  4. MIGRATION + HALO: owned particles that left the slab go to the neighbour
     (they move less than R per step, else an error), owned particles within R of a
     face go to that neighbour as ghosts, and each rank keeps its own emigrants as
     ghosts; the local set is rebuilt in place (nau_rebuild_rows: kept particles +
     arrivals, one pass) — no full reload;
  5. every `rebalance_every` steps the bounds are recomputed from the all-reduced
     x-histogram and owned particles hop rank by rank to their new owner.

Both ranks list a ghost in the same global cell grid ordered by global id, so the
ghost slots of a face and the owner's boundary slots run in the same order and the
halo values need no ids. Every neighbour sum runs over the present subset of the
single-GPU candidates in the single-GPU order (a missing candidate lies beyond R):
results are bitwise equal to one rank (tests/test_slab_gloo.py). x is a ring when
periodic (ghost positions stay true positions; periodic images do the rest). On one
rank there is nothing to exchange. The reference has no domain decomposition
(PAPER.md:152); this is new.

The rank logic is written against a small backend interface so it runs both on the
CUDA library (GpuBackend: device rows as torch tensors, NCCL) and, in the CPU tests,
on the oracle (tests/slab_oracle.py, gloo).
"""
from __future__ import annotations

import math

import numpy as np

FLAG_OWNED, FLAG_LEFT, FLAG_RIGHT = 0.0, 1.0, 2.0


def bounds_from_xhist(hist, x0: float, x1: float, world: int, min_width: float) -> list[float]:
    """Slab bounds [X_0 = x0, ..., X_world = x1] at histogram bin edges with ~equal
    counts; every slab at least `min_width` wide (2 R: a ghost never spans a slab)."""
    hist = np.asarray(hist, dtype=np.int64)
    nb = len(hist)
    edges = x0 + (x1 - x0) * np.arange(nb + 1) / nb
    cum = np.concatenate([[0], np.cumsum(hist)])
    total = int(cum[-1])
    bounds = [float(x0)]
    for r in range(1, world):
        i = int(np.searchsorted(cum, total * r / world, side="left"))
        b = float(edges[min(max(i, 0), nb)])
        lo_lim = bounds[-1] + min_width
        hi_lim = x1 - (world - r) * min_width
        bounds.append(min(max(b, lo_lim), hi_lim))
    bounds.append(float(x1))
    return bounds


def balanced_x_bounds(x, x0, x1, world, min_width, nbins=4096):
    """bounds_from_xhist from positions (the initial decomposition)."""
    h, _ = np.histogram(np.clip(x, x0, np.nextafter(x1, x0)), bins=nbins, range=(x0, x1))
    return bounds_from_xhist(h, x0, x1, world, min_width)


def owner_of(x, bounds):
    """Rank owning coordinate x (numpy, vectorised)."""
    return np.clip(np.searchsorted(np.asarray(bounds), x, side="right") - 1, 0, len(bounds) - 2)


def ghost_flags(x, bounds, rank, radius, periodic):
    """Flag of each particle for `rank`: 0 owned, 1 ghost owned by the left neighbour
    (within R below the left face), 2 by the right one (within R from the right face),
    -1 not present."""
    world = len(bounds) - 1
    x0, x1 = bounds[rank], bounds[rank + 1]
    ext = bounds[-1] - bounds[0]
    owned = (x >= x0) & (x < x1)
    flag = np.where(owned, FLAG_OWNED, -1.0)
    if world == 1:
        return flag
    if periodic:
        dl = np.mod(x0 - x, ext)
        dr = np.mod(x - x1, ext)
    else:
        dl = np.where(x < x0, x0 - x, np.inf)
        dr = np.where(x >= x1, x - x1, np.inf)
    left = ~owned & (dl > 0) & (dl <= radius) & (periodic or rank > 0)
    right = ~owned & (dr < radius) & (periodic or rank < world - 1)
    # a 2-rank ring has the same neighbour on both sides: the nearer face decides
    left_w = left & (~right | (dl <= dr))
    right_w = right & ~left_w
    flag = np.where(left_w, FLAG_LEFT, flag)
    return np.where(right_w, FLAG_RIGHT, flag)


def initial_rows(scene, field_names, bounds, rank, radius, periodic):
    """Host rows (owned + ghosts) of `rank` from the full scene; columns: r, fields...,
    gid, flag (0 owned, 1 ghost of the left neighbour, 2 of the right one)."""
    n = scene.n
    flag = ghost_flags(scene.pos[0], bounds, rank, radius, periodic)
    cols = [scene.pos]
    for name in field_names:
        cols.append(np.asarray(scene.fields[name], dtype=np.float64).reshape(-1, n))
    cols.append(np.arange(n, dtype=np.float64)[None, :])
    cols.append(flag[None, :])
    rows = np.concatenate(cols, axis=0).T
    return np.ascontiguousarray(rows[flag >= 0])


class Exchanger:
    """Variable-size row exchange with the left/right neighbours."""

    def __init__(self, dist, rank, world, periodic, device):
        self.dist, self.rank, self.world, self.periodic = dist, rank, world, periodic
        self.device = device
        self.left = (rank - 1) % world if (periodic or rank > 0) else None
        self.right = (rank + 1) % world if (periodic or rank < world - 1) else None

    def allreduce_sum(self, t):
        """Element-wise sum of a small tensor over the ranks (in place)."""
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
        # gloo moves P2P messages from host memory only: device rows are staged through
        # the host (multi-rank plumbing checks on a one-GPU box; NCCL sends device rows)
        staged = str(dev) != "cpu" and d.get_backend() == "gloo"
        out_dev = dev
        if staged:
            dev = "cpu"
            to_left = None if to_left is None else to_left.cpu()
            to_right = None if to_right is None else to_right.cpu()
        n_l = 0 if to_left is None else to_left.shape[0]
        n_r = 0 if to_right is None else to_right.shape[0]
        cnt_s = torch.tensor([n_l, n_r], dtype=torch.int64, device=dev)
        cnt_r = torch.zeros(2, dtype=torch.int64, device=dev)
        ops = []
        if self.left is not None:
            ops.append(d.P2POp(d.isend, cnt_s[0:1], self.left))
        if self.right is not None:
            ops.append(d.P2POp(d.isend, cnt_s[1:2], self.right))
            ops.append(d.P2POp(d.irecv, cnt_r[1:2], self.right))
        if self.left is not None:
            ops.append(d.P2POp(d.irecv, cnt_r[0:1], self.left))
        for w in d.batch_isend_irecv(ops):
            w.wait()
        counts = cnt_r.cpu()  # one device->host read for both counts
        from_left = torch.empty((int(counts[0]), width), dtype=torch.float64, device=dev)
        from_right = torch.empty((int(counts[1]), width), dtype=torch.float64, device=dev)
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
        if staged:
            from_left, from_right = from_left.to(out_dev), from_right.to(out_dev)
        return (from_left if self.left is not None else None,
                from_right if self.right is not None else None)


class SlabRank:
    """The per-rank driver. `backend` provides:
        width, col_gid, col_flag             row layout (col 0 = x)
        halo_values                          True for the two-pass WCSPH deck
        passes(k)                            k = "density" | "momentum" | "integrate" | "step"
        select_x(x_lo, x_hi, f_lo, f_hi)     slots of active particles with x in [x_lo, x_hi)
                                             and flag in [f_lo, f_hi], ascending slot order
        count(slots), pack(slots), pack_rho_p(slots)
        ghost_update(slots, rows)            (rho, p) into ghost slots
        rebuild(keep_slots, new_rows)        local set = kept slots + new rows (in place)
        hist_x(x0, x1, nbins)                per-bin counts of owned particles (tensor)
        with_flag(rows, f), cat(blocks), nrows(rows), x_of(rows), gid_of(rows),
        take(rows, mask)
    """

    def __init__(self, backend, exchanger, bounds, radius, periodic, rebalance_every=0,
                 nbins=4096):
        self.b = backend
        self.x = exchanger
        self.r = exchanger.rank
        self.bounds = [float(v) for v in bounds]
        self.R = float(radius)
        self.periodic = periodic
        self.ext = self.bounds[-1] - self.bounds[0]
        self.rebalance_every = rebalance_every
        self.nbins = nbins
        self.steps = 0
        self.rebalances = 0  # bound changes so far

    @property
    def lo_x(self):
        return self.bounds[self.r]

    @property
    def hi_x(self):
        return self.bounds[self.r + 1]

    # ---- one step ----
    def step(self):
        """One step of the §8(e) schedule. The backend's device work and the row tensors of
        the exchange must share one stream: the CUDA backend makes its context's stream
        torch's current stream for the whole step (`on_stream`), so a pack kernel and the
        NCCL send of its rows are ordered without host synchronisation."""
        import contextlib
        with getattr(self.b, "on_stream", contextlib.nullcontext)():
            self._step()

    def _step(self):
        b = self.b
        if b.halo_values and self.x.world > 1:
            b.passes("density")
            self.halo_values()
            b.passes("momentum")
            b.passes("integrate")
        else:
            b.passes("step")
        self.steps += 1
        if self.x.world == 1:
            return  # one rank owns everything: nothing to exchange
        if self.rebalance_every and self.steps % self.rebalance_every == 0:
            self.rebalance()
        else:
            self.exchange()

    def halo_values(self):
        """Step 2: (rho, p) of every owned particle within R of a face to that neighbour;
        ghosts of each face receive them in slot order (the same global order)."""
        b, X0, X1, R = self.b, self.lo_x, self.hi_x, self.R
        to_left = b.pack_rho_p(b.select_x(X0, X0 + R, FLAG_OWNED, FLAG_OWNED))
        to_right = b.pack_rho_p(b.select_x(X1 - R, X1, FLAG_OWNED, FLAG_OWNED))
        from_left, from_right = self.x.swap(to_left, to_right, 2)
        for blk, flag in ((from_left, FLAG_LEFT), (from_right, FLAG_RIGHT)):
            slots = b.select_x(-math.inf, math.inf, flag, flag)
            m = 0 if blk is None else blk.shape[0]
            if b.count(slots) != m:
                raise RuntimeError(f"slab halo values: {b.count(slots)} ghosts of flag {flag} "
                                   f"but {m} values received")
            if m:
                b.ghost_update(slots, blk)

    def _emigrants(self):
        """Owned particles that left [X0, X1): rows going left and right."""
        b, X0, X1 = self.b, self.lo_x, self.hi_x
        lo, hi = self.bounds[0], self.bounds[-1]
        out = b.cat([b.pack(b.select_x(lo, X0, FLAG_OWNED, FLAG_OWNED)),
                     b.pack(b.select_x(X1, hi, FLAG_OWNED, FLAG_OWNED))])
        x = b.x_of(out)
        if self.periodic:
            dl = np.mod(X0 - x, self.ext)
            dr = np.mod(x - X1, self.ext)
        else:
            dl = np.where(x < X0, X0 - x, np.inf)
            dr = np.where(x >= X1, x - X1, np.inf)
        go_left = dl <= dr
        far = np.minimum(dl, dr) >= self.R
        if np.any(far):
            g = b.gid_of(out)[far]
            raise RuntimeError(f"slab migration: particle(s) {g[:5].tolist()} moved more than the "
                               f"interaction radius past the slab face in one step")
        if (self.x.left is None and np.any(go_left)) or (self.x.right is None and np.any(~go_left)):
            raise RuntimeError("slab migration: a particle left the outermost slab")
        return b.take(out, go_left), b.take(out, ~go_left)

    def exchange(self):
        """Step 4: migration and the ghost halo in one exchange round, rebuilt in place."""
        b, X0, X1, R = self.b, self.lo_x, self.hi_x, self.R
        em_l, em_r = self._emigrants()
        keep = b.select_x(X0, X1, FLAG_OWNED, FLAG_OWNED)
        bnd_l = b.pack(b.select_x(X0, X0 + R, FLAG_OWNED, FLAG_OWNED))
        bnd_r = b.pack(b.select_x(X1 - R, X1, FLAG_OWNED, FLAG_OWNED))
        to_left = b.cat([em_l, b.with_flag(bnd_l, FLAG_RIGHT)])   # the left rank's right ghosts
        to_right = b.cat([em_r, b.with_flag(bnd_r, FLAG_LEFT)])
        from_left, from_right = self.x.swap(to_left, to_right, b.width)
        # emigrants stay here as ghosts of the rank that now owns them
        b.rebuild(keep, b.cat([from_left, from_right, b.with_flag(em_l, FLAG_LEFT),
                               b.with_flag(em_r, FLAG_RIGHT)]))

    def rebalance(self):
        """Step 5: new bounds from the all-reduced x-histogram of owned particles; owned
        particles hop rank by rank toward their new owner (nearer direction on a ring),
        then the ghost halo is rebuilt for the new faces."""
        import torch
        b = self.b
        lo, hi = self.bounds[0], self.bounds[-1]
        b.rebuild(b.select_x(lo, hi, FLAG_OWNED, FLAG_OWNED), None)  # drop the ghosts
        hist = self.x.allreduce_sum(b.hist_x(lo, hi, self.nbins))
        total = int(hist.sum().item())
        new = bounds_from_xhist(hist.cpu().numpy(), lo, hi, self.x.world, 2.0 * self.R)
        if new != self.bounds:
            self.bounds = new
            self.rebalances += 1
        W, me = self.x.world, self.r
        for _ in range(W + 1):
            rows = b.cat([b.pack(b.select_x(lo, self.lo_x, FLAG_OWNED, FLAG_OWNED)),
                          b.pack(b.select_x(self.hi_x, hi, FLAG_OWNED, FLAG_OWNED))])
            own = owner_of(b.x_of(rows), self.bounds)
            if self.periodic:
                right = np.mod(own - me, W) <= W // 2
            else:
                right = own > me
            cnt = torch.tensor([b.nrows(rows)], dtype=torch.int64, device=self.x.device)
            if int(self.x.allreduce_sum(cnt).item()) == 0:
                break
            keep = b.select_x(self.lo_x, self.hi_x, FLAG_OWNED, FLAG_OWNED)
            from_left, from_right = self.x.swap(b.take(rows, ~right), b.take(rows, right),
                                                b.width)
            b.rebuild(keep, b.cat([from_left, from_right]))
        else:
            raise RuntimeError("slab rebalance: particles still misplaced after world+1 hops")
        got = torch.tensor([b.count(b.select_x(lo, hi, FLAG_OWNED, FLAG_OWNED))],
                           dtype=torch.int64, device=self.x.device)
        if int(self.x.allreduce_sum(got).item()) != total:  # duplicated or dropped in transit
            raise RuntimeError(f"slab rebalance: {int(got.item())} owned rows after the hops, "
                               f"{total} before")
        X0, X1, R = self.lo_x, self.hi_x, self.R
        keep = b.select_x(X0, X1, FLAG_OWNED, FLAG_OWNED)
        bnd_l = b.pack(b.select_x(X0, X0 + R, FLAG_OWNED, FLAG_OWNED))
        bnd_r = b.pack(b.select_x(X1 - R, X1, FLAG_OWNED, FLAG_OWNED))
        from_left, from_right = self.x.swap(b.with_flag(bnd_l, FLAG_RIGHT),
                                            b.with_flag(bnd_r, FLAG_LEFT), b.width)
        b.rebuild(keep, b.cat([from_left, from_right]))


class GpuBackend:
    """Backend over the CUDA library; slots and rows are device tensors (torch)."""

    def __init__(self, ctx, wcsph_params=None, step_fn=None, gid_name="gid", flag_name="ghost"):
        import torch
        self.torch = torch
        self.ctx = ctx
        self.p = wcsph_params
        self.step_fn = step_fn
        self.halo_values = wcsph_params is not None and step_fn is None
        self.gid = ctx.fields[gid_name].id
        self.flag_id = ctx.fields[flag_name].id
        self.width = ctx.L.nau_row_width(ctx.h)
        self.col_gid = self.width - 2
        self.col_flag = self.width - 1
        self.device = f"cuda:{torch.cuda.current_device()}"
        ctx._check(ctx.L.nau_set_ghost_field(ctx.h, self.flag_id))

    def on_stream(self):
        """torch's current stream := the context's stream (row tensors, NCCL and the
        library's kernels then run in one order)."""
        torch = self.torch
        return torch.cuda.stream(torch.cuda.ExternalStream(self.ctx.L.nau_get_stream(self.ctx.h)))

    # ---- passes ----
    def passes(self, k):
        ctx = self.ctx
        if k == "step":
            if self.step_fn is not None:
                self.step_fn()
            else:
                ctx.wcsph_step(self.p)
        else:
            ctx.wcsph_pass(self.p, {"density": 0, "momentum": 1, "integrate": 2}[k])

    # ---- selections and rows ----
    def select_x(self, x0, x1, f0, f1):
        import ctypes as C
        torch = self.torch
        slots = torch.empty(max(1, self.ctx.n), dtype=torch.int32, device=self.device)
        cnt = C.c_long(0)
        self.ctx._check(self.ctx.L.nau_select_x(self.ctx.h, 0, float(x0), float(x1), self.flag_id,
                                                float(f0), float(f1), slots.data_ptr(),
                                                C.byref(cnt)))
        return slots[: cnt.value]

    def count(self, slots):
        return int(slots.shape[0])

    def pack(self, slots):
        m = int(slots.shape[0])
        rows = self.torch.empty((m, self.width), dtype=self.torch.float64, device=self.device)
        if m:
            self.ctx._check(self.ctx.L.nau_pack_rows(self.ctx.h, slots.data_ptr(), m,
                                                     rows.data_ptr()))
        return rows

    def pack_rho_p(self, slots):
        import ctypes as C
        m = int(slots.shape[0])
        rows = self.torch.empty((m, 2), dtype=self.torch.float64, device=self.device)
        if m:
            self.ctx._check(self.ctx.L.nau_wcsph_pack_rho_p(self.ctx.h, C.byref(self.p),
                                                            slots.data_ptr(), m, rows.data_ptr()))
        return rows

    def ghost_update(self, slots, rows):
        import ctypes as C
        rows = rows.contiguous()
        self.ctx._check(self.ctx.L.nau_wcsph_ghost_update(self.ctx.h, C.byref(self.p),
                                                          slots.data_ptr(), int(slots.shape[0]),
                                                          rows.data_ptr()))

    def rebuild(self, keep, rows):
        mk = int(keep.shape[0])
        rows = rows.contiguous() if rows is not None and rows.shape[0] else None
        mn = 0 if rows is None else int(rows.shape[0])
        self.ctx._check(self.ctx.L.nau_rebuild_rows(self.ctx.h, keep.data_ptr() if mk else None,
                                                    mk, rows.data_ptr() if mn else None, mn,
                                                    self.gid))
        self.ctx.n = mk + mn
        self._keep = (keep, rows)  # the copies run on the context stream

    def load(self, rows):
        rows = rows.contiguous()
        self.ctx._check(self.ctx.L.nau_load_rows(self.ctx.h, rows.data_ptr(), rows.shape[0],
                                                 self.gid))
        self.ctx.n = rows.shape[0]
        self._keep = rows

    def hist_x(self, x0, x1, nbins):
        h = self.torch.zeros(nbins, dtype=self.torch.int64, device=self.device)
        self.ctx._check(self.ctx.L.nau_histogram_x(self.ctx.h, 0, float(x0), float(x1), nbins,
                                                   self.flag_id, 0.0, 0.0, h.data_ptr()))
        self.ctx.sync()
        return h

    # ---- row helpers ----
    def with_flag(self, rows, f):
        if rows is None or rows.shape[0] == 0:
            return rows
        rows = rows.clone()
        rows[:, self.col_flag] = f
        return rows

    def cat(self, blocks):
        blocks = [b for b in blocks if b is not None and b.shape[0]]
        if not blocks:
            return self.torch.empty((0, self.width), dtype=self.torch.float64, device=self.device)
        return self.torch.cat(blocks, 0)

    def nrows(self, rows):
        return 0 if rows is None else int(rows.shape[0])

    def x_of(self, rows):
        return rows[:, 0].cpu().numpy()

    def gid_of(self, rows):
        return rows[:, self.col_gid].cpu().numpy().astype(np.int64)

    def take(self, rows, mask):
        return rows[self.torch.as_tensor(np.asarray(mask, bool), device=rows.device)]


# ------------------------------------------------------- sharded n-body sources ----
def pipelined_sources(dist, local_rows, bufs, world: int, rank: int, consume, wait=None):
    """Sharded all-pairs schedule: instead of one all-gather
    followed by the whole pair loop, rank c broadcasts its (x, y, z, m) rows as chunk c
    while every rank evaluates chunk c - 1 — the transfer of each chunk hides behind the
    pair loop over the previous one. Chunks are consumed in GLOBAL order 0..world-1 on
    every rank (`consume(c, rows)`, which continues the sums: nau_gravity_sources_part),
    so the result equals the single-GPU sum order bit for bit.

    `bufs`: two receive tensors shaped like `local_rows`; the broadcasts are asynchronous
    (`async_op=True`), `wait(work)` orders the consumer's stream after a transfer
    (default: work.wait(), which NCCL turns into a stream dependency, not a host block).
    """
    wait = wait or (lambda w: w.wait())

    def post(c):
        t = local_rows if c == rank else bufs[c & 1]
        return t, dist.broadcast(t, src=c, async_op=True)

    nxt = post(0)
    for c in range(world):
        rows, work = nxt
        wait(work)
        if c + 1 < world:
            nxt = post(c + 1)  # lands in the other buffer while chunk c is evaluated
        consume(c, rows)
