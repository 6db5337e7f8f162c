"""TEST INFRASTRUCTURE: a SlabRank backend on the oracle (oracle/port + the deck
restatement in tests/deck_oracle.py), so the multi-rank slab logic of
paper_1710_08259_b200/slab.py runs on CPU under gloo. Rows are torch CPU tensors
with the GpuBackend layout: r, rho, p, v, vdot, mask, gid, flag; slots are row
indices. Like the device path, the rows are put in (cell, global id) order by each
density pass (the cell build), so halo values are matched in slot order.
"""
from __future__ import annotations

import numpy as np
import torch

import deck_oracle
from oracle import port

FIELDS = ["rho", "p", "v", "vdot", "mask"]


class OracleBackend:
    halo_values = True

    def __init__(self, scene):
        self.sc = scene
        self.prm = scene.params
        self.dim = scene.dim
        d = self.dim
        self.width = d + 1 + 1 + d + d + 1 + 2
        self.col_gid = self.width - 2
        self.col_flag = self.width - 1
        self.dom = port.Domain(scene.dim, scene.min_cells, scene.max_cells, scene.cell_size,
                               scene.kinds)
        self.rows = np.zeros((0, self.width))
        self.active = np.zeros(0, bool)
        self.ps = None

    # ---- state ----
    def load(self, rows):
        r = rows.numpy() if isinstance(rows, torch.Tensor) else np.asarray(rows)
        self.rows = np.ascontiguousarray(r.copy())
        self.active = np.ones(len(self.rows), bool)
        self.ps = None

    def _split(self):
        d, r = self.dim, self.rows.T
        o = d
        st = {}
        for name, w in (("rho", 1), ("p", 1), ("v", d), ("vdot", d), ("mask", 1)):
            st[name] = np.ascontiguousarray(r[o:o + w])
            o += w
        return np.ascontiguousarray(r[:d]), st

    def _store(self, st):
        cols = [self.ps.pos] + [st[k] for k in FIELDS]
        self.rows[:, :self.col_gid] = np.concatenate(cols, axis=0).T
        self.active = self.ps.active.astype(bool)

    def _build(self):
        """The cell build: rows in (flat cell, global id) order, inactive last."""
        pos, _ = self._split()
        ps = port.ParticleSystem(self.dom, pos, self.active.astype(np.uint8))
        cell_of = ps.build_cells()[0]
        key = np.where(cell_of >= 0, cell_of, np.iinfo(np.int32).max).astype(np.int64)
        order = np.lexsort((self.rows[:, self.col_gid], key))
        self.rows = np.ascontiguousarray(self.rows[order])
        self.active = self.active[order]
        pos, st = self._split()
        self.ps = port.ParticleSystem(self.dom, pos, self.active.astype(np.uint8))
        self.ps.build_cells()
        return st

    # ---- passes ----
    def passes(self, k):
        if k == "step":
            st = self._build()
            deck_oracle.step(self.ps, st, self.prm)
            self._store(st)
        elif k == "density":
            st = self._build()
            deck_oracle.density(self.ps, st, self.prm)
            self._store(st)
        elif k == "momentum":
            _, st = self._split()
            deck_oracle.momentum(self.ps, st, self.prm)
            self._store(st)
        else:
            _, st = self._split()
            deck_oracle.integrate(self.ps, st, self.prm, upd=self.rows[:, self.col_flag] == 0)
            self._store(st)

    # ---- selections and rows ----
    def select_x(self, x0, x1, f0, f1):
        x, f = self.rows[:, 0], self.rows[:, self.col_flag]
        m = self.active & (x >= x0) & (x < x1) & (f >= f0) & (f <= f1)
        return np.flatnonzero(m)

    def count(self, slots):
        return len(slots)

    def pack(self, slots):
        return torch.from_numpy(self.rows[slots].copy())

    def pack_rho_p(self, slots):
        d = self.dim
        return torch.from_numpy(self.rows[slots][:, [d, d + 1]].copy())

    def ghost_update(self, slots, rows):
        d = self.dim
        r = rows.numpy()
        self.rows[slots, d] = r[:, 0]
        self.rows[slots, d + 1] = r[:, 1]

    def rebuild(self, keep, rows):
        blocks = [self.rows[keep]]
        act = [self.active[keep]]
        if rows is not None and rows.shape[0]:
            blocks.append(rows.numpy())
            act.append(np.ones(rows.shape[0], bool))
        self.rows = np.ascontiguousarray(np.concatenate(blocks, axis=0))
        self.active = np.concatenate(act)
        self.ps = None

    def hist_x(self, x0, x1, nbins):
        m = self.active & (self.rows[:, self.col_flag] == 0)
        x = self.rows[m, 0]
        b = np.clip(np.floor((x - x0) * (nbins / (x1 - x0))).astype(np.int64), 0, nbins - 1)
        return torch.from_numpy(np.bincount(b, minlength=nbins).astype(np.int64))

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
            return torch.zeros((0, self.width), dtype=torch.float64)
        return torch.cat(blocks, 0)

    def nrows(self, rows):
        return 0 if rows is None else int(rows.shape[0])

    def x_of(self, rows):
        return rows[:, 0].numpy()

    def gid_of(self, rows):
        return rows[:, self.col_gid].numpy().astype(np.int64)

    def take(self, rows, mask):
        return rows[torch.from_numpy(np.asarray(mask, bool))]

    def owned(self):
        m = self.active & (self.rows[:, self.col_flag] == 0)
        return self.rows[m]
