"""FAST against EXACT over a longer run than the 10 steps the parity tests cover: the cfg2
geometry at dx = 0.02, both modes from the same state, relative field differences and
conserved quantities every 25 steps.

    python tools/mode_drift.py --steps 200
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1710_08259_b200 import nau, scenes  # noqa: E402


def make(sc, fast):
    prm = sc.params
    c = nau.Context(0)
    c.set_mode(fast)
    c.set_domain(sc.dim, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
    c.set_particles(sc.pos)
    for k in ("rho", "p", "v", "vdot", "mask"):
        v = np.asarray(sc.fields[k]).reshape(-1, sc.n)
        c.add_field(k, v.shape[0], 1, v)
    c.boundary_shift()
    p = nau.WcsphParams()
    p.kernel_family, p.kernel_dim = nau.K_WENDLAND, 3
    p.mass, p.radius, p.rho0, p.B = prm["mass"], prm["radius"], prm["rho0"], prm["B"]
    p.gamma, p.visc, p.dt = prm["gamma"], prm["visc"], prm["dt"]
    for ax in range(3):
        p.g[ax] = prm["g"][ax]
    f = c.fields
    p.f_rho, p.f_p, p.f_v, p.f_vdot, p.f_mask = f["rho"].id, f["p"].id, f["v"].id, f["vdot"].id, f["mask"].id
    return c, p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--dx", type=float, default=0.02)
    a = ap.parse_args()
    sc = scenes.dam_break(3, dx=a.dx)
    (ce, pe), (cf, pf) = make(sc, False), make(sc, True)
    nf = sc.params["n_fluid"]
    for s in range(25, a.steps + 1, 25):
        for _ in range(25):
            ce.wcsph_step(pe)
            cf.wcsph_step(pf)
        ce.sync(); cf.sync()
        row = {"step": s}
        for k in ("r", "v", "rho"):
            e, f = ce.download(k), cf.download(k)
            row[k] = float(np.abs(e - f).max() / max(np.abs(e).max(), 1e-300))
        ve, vf = ce.download("v")[:, :nf], cf.download("v")[:, :nf]
        row["ke_rel"] = float(abs((ve ** 2).sum() - (vf ** 2).sum()) / max((ve ** 2).sum(), 1e-300))
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
