"""Robustness run: a 3D dam break collapsing for thousands of steps in FAST mode (graph
replay, async lists). Reports particle count, kinetic energy, max speed, density range,
list shape and ms/step along the way — cells fill past the lattice count as the column
collapses (more list blocks, capacity growth, overflow fallback).

    python tools/long_run.py --dx 0.01 --steps 4000 --every 500
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_1710_08259_b200 import nau, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dx", type=float, default=0.01)
    ap.add_argument("--steps", type=int, default=4000)
    ap.add_argument("--every", type=int, default=500)
    ap.add_argument("--mode", default="fast")
    a = ap.parse_args()
    sc = scenes.dam_break(3, dx=a.dx)
    prm = sc.params
    c = nau.Context(0)
    c.set_mode(a.mode == "fast")
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
    nf = prm["n_fluid"]
    done = 0
    while done < a.steps:
        t0 = time.perf_counter()
        for _ in range(a.every):
            c.wcsph_step(p)
        c.sync()
        ms = (time.perf_counter() - t0) * 1e3 / a.every
        done += a.every
        v, rho, r = c.download("v"), c.download("rho")[0], c.download("r")
        c.wcsph_pass(p, 0)
        st = c.list_stats()
        row = {"step": done, "t": round(done * prm["dt"], 4), "ms_per_step": round(ms, 3),
               "active": int(c.active().sum()), "warnings": int(c.warning_count() if callable(c.warning_count) else c.warning_count),
               "ke": float(0.5 * prm["mass"] * (v[:, :nf] ** 2).sum()),
               "vmax": float(np.sqrt((v ** 2).sum(0)).max()),
               "rho_min": float(rho[:nf].min()), "rho_max": float(rho[:nf].max()),
               "x_front": float(r[0, :nf].max()),
               "entries_per_walker": round(st["entries_per_walker"], 1),
               "lane_eff": round(st["lane_efficiency"], 3)}
        print(json.dumps(row), flush=True)
        assert np.isfinite(v).all() and np.isfinite(rho).all()
    # per-kernel times in the evolved state (launch events; plain steps)
    c.profile(True)
    for _ in range(5):
        c.wcsph_step(p)
    c.sync()
    names = {300: "cell build", 302: "list build", 200: "density", 201: "momentum", 301: "symplectic"}
    print(json.dumps({"evolved_ms": {v: round(c.profile_ms(k)[0] / max(c.profile_ms(k)[1], 1), 4)
                                     for k, v in names.items()}}), flush=True)
    c.close()


if __name__ == "__main__":
    main()
