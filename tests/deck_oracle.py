"""TEST INFRASTRUCTURE: the BASELINE WCSPH deck stepped with the C port
(oracle/port), equation by equation in the reference's order and arithmetic
(scenes.wcsph_equations; src/case.cpp:9-67). Pinned against the reference's
own Case::solve_step in tests/test_oracle.py.
"""
from __future__ import annotations

import math

import numpy as np

from oracle import port


def make_system(scene):
    dom = port.Domain(scene.dim, scene.min_cells, scene.max_cells, scene.cell_size, scene.kinds)
    ps = port.ParticleSystem(dom, scene.pos)
    ps.boundary_shift()
    ps.build_cells()
    st = {k: np.array(v, dtype=np.float64).reshape(-1, scene.n).copy()
          for k, v in scene.fields.items()}
    return ps, st


def density(ps, st, prm, kfamily=port.K_WENDLAND):
    """rho = sph_S(one, mass, one, K, R); p = B*((rho/rho0)^gam - 1)."""
    dim = ps.dom.dim
    act = ps.active.astype(bool)
    R, m = prm["radius"], prm["mass"]
    if ps.tables is None:
        ps.build_cells()
    rho = ps.interact(port.SPH_S, [1.0, m, 1.0, R], (1, 1), kfamily=kfamily, kdim=dim,
                      init=st["rho"])
    st["rho"] = rho
    p = st["p"].copy()
    # libm pow per element (numpy's SIMD power differs from glibc pow by an ulp)
    ratio = rho[0, act] / prm["rho0"]
    powed = np.array([math.pow(x, prm["gamma"]) for x in ratio.tolist()], dtype=np.float64)
    p[0, act] = prm["B"] * (powed - 1.0)
    st["p"] = p
    return st


def momentum(ps, st, prm, kfamily=port.K_WENDLAND):
    """vdot = -1/rho*sph_G11(p, mass, rho, K, R) + visc*sph_A(v, mass, rho, K, R) + g."""
    dim = ps.dom.dim
    act = ps.active.astype(bool)
    R, m = prm["radius"], prm["mass"]
    rho = st["rho"]
    G = ps.interact(port.SPH_G11, [st["p"], m, rho, R], (dim, 1), kfamily=kfamily, kdim=dim)
    A = ps.interact(port.SPH_A, [st["v"], m, rho, R], (dim, 1), kfamily=kfamily, kdim=dim)
    g = np.asarray(prm["g"], dtype=np.float64).reshape(dim, 1)
    vdot = st["vdot"].copy()
    vdot[:, act] = ((-1.0 / rho[:, act]) * G[:, act] + prm["visc"] * A[:, act]) + g
    st["vdot"] = vdot
    return st


def integrate(ps, st, prm, upd=None):
    """v = euler(v, vdot*mask, dt); r = euler(r, v, dt); boundary shift. upd: the particles
    updated (slab ghosts are not)."""
    act = ps.active.astype(bool)
    if upd is not None:
        act = act & upd
    v = st["v"].copy()
    v[:, act] = v[:, act] + prm["dt"] * (st["mask"][:, act] * st["vdot"][:, act])
    st["v"] = v
    pos = ps.pos
    pos[:, act] = pos[:, act] + prm["dt"] * v[:, act]
    ps.boundary_shift()  # case.cpp:59-62, then dirty
    ps.tables = None
    return st


def step(ps, st, prm, kfamily=port.K_WENDLAND):
    """One solve_step of the deck; mutates ps (positions/active/cells) and st."""
    density(ps, st, prm, kfamily)
    momentum(ps, st, prm, kfamily)
    return integrate(ps, st, prm)
