"""TEST INFRASTRUCTURE: a SlabRank backend on the oracle (oracle/port + the deck
restatement in tests/deck_oracle.py), so the multi-rank slab logic of
paper_1710_08259_b200/slab.py runs on CPU under gloo. Rows are torch CPU tensors
with the GpuBackend layout: r, rho, p, v, vdot, mask, gid, ghost.
"""
from __future__ import annotations

import numpy as np
import torch

import deck_oracle
from oracle import port
from paper_1710_08259_b200.slab import cell_x_of

FIELDS = ["rho", "p", "v", "vdot", "mask"]


class OracleBackend:
    def __init__(self, scene, ncx, periodic):
        self.sc = scene
        self.prm = scene.params
        self.dim = scene.dim
        d = self.dim
        self.width = d + 1 + 1 + d + d + 1 + 2
        self.col_gid = self.width - 2
        self.col_ghost = self.width - 1
        self.ncx, self.periodic = ncx, periodic
        self.lo = scene.min_cells[0] * scene.cell_size[0]
        self.cs = scene.cell_size[0]
        self.rows = np.zeros((0, self.width))
        self.active = np.zeros(0, bool)

    def load(self, rows):
        r = rows.numpy() if isinstance(rows, torch.Tensor) else np.asarray(rows)
        order = np.argsort(r[:, self.col_gid], kind="stable")  # cells list ascending gid
        self.rows = np.ascontiguousarray(r[order])
        self.active = np.ones(len(self.rows), bool)

    def select(self, c0, c1, ghost):
        cx = cell_x_of(self.rows[:, 0], self.lo, self.cs, self.ncx, self.periodic)
        m = self.active & (cx >= c0) & (cx < c1) & (self.rows[:, self.col_ghost] == ghost)
        return torch.from_numpy(self.rows[m].copy())

    def mark_ghost(self, rows):
        rows = rows.clone()
        rows[:, self.col_ghost] = 1.0
        return rows

    def cat(self, blocks):
        blocks = [b for b in blocks if b is not None and b.shape[0]]
        if not blocks:
            return torch.zeros((0, self.width), dtype=torch.float64)
        return torch.cat(blocks, 0)

    def _split(self):
        d, r = self.dim, self.rows.T
        o = d
        st = {}
        for name, w in (("rho", 1), ("p", 1), ("v", d), ("vdot", d), ("mask", 1)):
            st[name] = np.ascontiguousarray(r[o:o + w])
            o += w
        return np.ascontiguousarray(r[:d]), st

    def step(self):
        sc = self.sc
        pos, st = self._split()
        dom = port.Domain(sc.dim, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
        ps = port.ParticleSystem(dom, pos, self.active.astype(np.uint8))
        ps.build_cells()
        deck_oracle.step(ps, st, self.prm)
        d = self.dim
        cols = [ps.pos] + [st[k] for k in FIELDS]
        self.rows[:, :self.col_gid] = np.concatenate(cols, axis=0).T
        self.active = ps.active.astype(bool)
