"""TEST INFRASTRUCTURE: conserved and balance quantities of the BASELINE decks,
computed identically (numpy, index order) from the GPU's and the oracle's fields,
so a comparison measures only the difference between the two states.

north_star: "Multi-step runs must agree on conserved quantities (mass exactly;
momentum and energy within 1e-8 relative)". The reference pins its own
conservation properties in tests/acceptance/acceptance.cpp:341-394 (fsum per
step, sph_G11 pairwise momentum) and tests/test_interactions.cpp:384-406 (orbit
energy within 1%).
"""
from __future__ import annotations

import numpy as np


def wcsph_energy(pos, v, rho, active, prm):
    """Components of the WCSPH deck's total energy over active particles:
    kinetic 1/2 m|v|^2, gravitational -m g.r, and the Tait internal energy
    m u(rho) with u = int_{rho0}^{rho} p/rho'^2 drho' for p = B((rho/rho0)^gam - 1):
    u = B [ (rho^(gam-1)/rho0^gam - 1/rho0)/(gam-1) + 1/rho - 1/rho0 ]."""
    act = np.asarray(active).astype(bool)
    m, B, r0, gam = prm["mass"], prm["B"], prm["rho0"], prm["gamma"]
    g = np.asarray(prm["g"], np.float64).reshape(-1, 1)
    ke = 0.5 * m * float((v[:, act] ** 2).sum())
    pe = -m * float((g * pos[:, act]).sum())
    rr = rho.reshape(-1)[act]
    u = B * ((rr ** (gam - 1.0) / r0 ** gam - 1.0 / r0) / (gam - 1.0) + 1.0 / rr - 1.0 / r0)
    ie = m * float(u.sum())
    return {"kinetic": ke, "gravitational": pe, "internal": ie, "total": ke + pe + ie}


def momentum(v, mass, active):
    """Total momentum per axis and its scale (sum of m|v|, the magnitude a relative
    comparison is taken against when the total itself is ~0)."""
    act = np.asarray(active).astype(bool)
    m = np.broadcast_to(np.asarray(mass, np.float64).reshape(-1), act.shape)[act]
    mv = v[:, act] * m
    return mv.sum(axis=1), float(np.sqrt((mv ** 2).sum(axis=0)).sum())


def dem_energy(pos, v, mass, g, active):
    """Kinetic + gravitational energy of the granular column (the contact springs'
    stored energy is not a field of the deck)."""
    act = np.asarray(active).astype(bool)
    m = np.asarray(mass, np.float64).reshape(-1)[act]
    ke = 0.5 * float((m * (v[:, act] ** 2).sum(axis=0)).sum())
    pe = -float((m * (np.asarray(g, np.float64).reshape(-1, 1) * pos[:, act]).sum(axis=0)).sum())
    return {"kinetic": ke, "gravitational": pe, "total": ke + pe}


def nbody_energy(pos, v, m, G, eps, chunk=1024):
    """Kinetic + Plummer-softened potential -sum_{i<j} G m^2 / sqrt(r^2 + eps^2)."""
    n = pos.shape[1]
    ke = 0.5 * m * float((v ** 2).sum())
    pe = 0.0
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        d = pos[:, s:e, None] - pos[:, None, :]
        r = np.sqrt((d ** 2).sum(axis=0) + eps * eps)
        inv = 1.0 / r
        idx = np.arange(s, e)
        inv[idx - s, idx] = 0.0
        pe -= 0.5 * G * m * m * float(inv.sum())
    return {"kinetic": ke, "potential": pe, "total": ke + pe}


def assert_agree(got: dict, exp: dict, tol: float, what: str):
    """Every component within tol relative to its own magnitude (and the total)."""
    for k in exp:
        scale = max(abs(exp[k]), 1e-300)
        err = abs(got[k] - exp[k]) / scale
        assert err <= tol, f"{what} {k}: {got[k]!r} vs {exp[k]!r} (rel {err:.3e} > {tol})"
