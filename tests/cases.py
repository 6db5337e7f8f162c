"""Shared parity cases: one spec drives the reference (oracle/_ref), the C port
(oracle/port) and the CUDA path (paper_1710_08259_b200.nau).

A spec is a dict: dim, min_cells, max_cells, cell_size, kinds, pos (dim, n),
fields {name: (comps, n)}, consts {name: value}. Operators are written the
reference's way, e.g. ("sph_G11", ["A", "m", "rho", "R"], "Wp53220").
"""
from __future__ import annotations

import numpy as np

SPH_OPS = ["sph_S", "sph_D00", "sph_G11", "sph_L0", "sph_A"]


def random_spec(rng, dim=None, n=None, kinds=None, cells=None, cs=0.3):
    dim = int(dim or rng.integers(1, 4))
    kinds = list(kinds if kinds is not None else rng.integers(0, 3, size=dim))
    cells = list(cells if cells is not None else rng.integers(1, 6, size=dim))
    n = int(n if n is not None else rng.integers(1, 160))
    lo = [0.0] * dim
    hi = [c * cs for c in cells]
    pos = np.stack([rng.uniform(lo[a], hi[a], n) for a in range(dim)]) if n else np.zeros((dim, 0))
    R = cs
    return {
        "dim": dim, "min_cells": [0] * dim, "max_cells": cells, "cell_size": [cs] * dim,
        "kinds": kinds, "pos": np.ascontiguousarray(pos),
        "fields": {
            "A": rng.uniform(0.0, 1.0, (1, n)),
            "V": rng.uniform(-1.0, 1.0, (dim, n)),
            "rho": rng.uniform(900.0, 1100.0, (1, n)),
            "M": rng.uniform(0.5, 1.5, (1, n)),
            "Rp": rng.uniform(0.05, 0.15, (1, n)),
        },
        "consts": {"m": 0.5, "R": R, "E": 2.06e6, "nu": 0.33, "kn": 1e5, "en": 0.5, "cf": 0.5,
                   "cf0": 0.0, "G": 1.0, "eps": 0.01, "Rs": R,
                   # sfm (social force) parameters: desired speed, repulsion A/B,
                   # body stiffness, attraction c, relaxation time
                   "sv0": 1.3, "sA": 2.0, "sB": 0.08, "sK": 120.0, "sC": 0.05, "stau": 0.5},
    }


def op_list(dim):
    """(name, operands, keyword|None, out_comps, port_op, port_kfamily)."""
    from oracle import port
    W, Cb = f"Wp5{dim}220", f"Wc3{dim}220"
    out = []
    for kw, fam in ((W, port.K_WENDLAND), (Cb, port.K_CUBIC)):
        out += [
            ("sph_S", ["A", "m", "rho", "R"], kw, 1, port.SPH_S, fam),
            ("sph_S", ["V", "M", "rho", "R"], kw, dim, port.SPH_S, fam),
            ("sph_G11", ["A", "m", "rho", "R"], kw, dim, port.SPH_G11, fam),
            ("sph_L0", ["A", "M", "rho", "R"], kw, 1, port.SPH_L0, fam),
            ("sph_A", ["V", "m", "rho", "R"], kw, dim, port.SPH_A, fam),
        ]
        if dim > 1:
            out.append(("sph_D00", ["V", "m", "rho", "R"], kw, 1, port.SPH_D00, fam))
    out += [
        ("dem_l", ["V", "Rp", "E", "nu", "M", "cf", "Rs"], None, dim, port.DEM_HERTZ, 0),
        ("dem_boundary_force", ["V", "Rp", "E", "nu", "M", "cf0", "Rs"], None, dim,
         port.DEM_BOUNDARY, 0),
        ("dem_lsd", ["V", "Rp", "kn", "en", "M", "cf", "Rs"], None, dim, port.DEM_LSD, 0),
        ("nbody_gravity", ["M", "G", "eps"], None, dim, port.GRAVITY, 0),
        # r_d = V: the desired positions are any d-vector field
        ("sfm", ["V", "sv0", "V", "Rp", "sA", "sB", "sK", "sC", "M", "stau"], None, dim,
         port.SFM, 0),
    ]
    return out


# ---------------------------------------------------------------- port ----
def port_system(spec):
    from oracle import port
    dom = port.Domain(spec["dim"], spec["min_cells"], spec["max_cells"], spec["cell_size"],
                      spec["kinds"])
    ps = port.ParticleSystem(dom, spec["pos"])
    ps.boundary_shift()
    ps.build_cells()
    return ps


def port_operand(spec, name):
    if name in spec["fields"]:
        return spec["fields"][name]
    return float(spec["consts"][name])


def port_eval(spec, ps, entry):
    name, operands, kw, comps, pop, fam = entry
    kdim = int(kw[3]) if kw else None
    return ps.interact(pop, [port_operand(spec, o) for o in operands], (comps, 1), kfamily=fam,
                       kdim=kdim)


# ----------------------------------------------------------------- ref ----
def ref_case(spec, seed=0):
    from oracle import ref
    rc = ref.RefCase(spec["dim"], spec["min_cells"], spec["max_cells"], spec["cell_size"],
                     spec["kinds"], spec["pos"], seed=seed)
    for k, v in spec["fields"].items():
        rc.field(k, v)
    for k, v in spec["consts"].items():
        rc.constant(k, float(v))
    return rc


def ref_eval(spec, rc, entry):
    name, operands, kw, comps, pop, fam = entry
    if name == "dem_lsd" or (kw is not None and kw[1] == "c"):
        return rc.eval_law(name, operands, comps, kdim=int(kw[3]) if kw else None)
    args = operands if kw is None else operands[:3] + [kw] + operands[3:]
    return rc.eval(f"{name}({','.join(args)})", comps)


# ----------------------------------------------------------------- gpu ----
def gpu_context(spec, ctx=None):
    from paper_1710_08259_b200 import nau
    ctx = ctx or nau.Context(0)
    ctx.set_domain(spec["dim"], spec["min_cells"], spec["max_cells"], spec["cell_size"],
                   spec["kinds"])
    ctx.set_particles(spec["pos"])
    for k, v in spec["fields"].items():
        v = np.atleast_2d(np.asarray(v))
        ctx.add_field(k, v.shape[0], 1, v)
    ctx.boundary_shift()
    ctx.build_cells()
    return ctx


def gpu_eval(spec, ctx, entry):
    name, operands, kw, comps, pop, fam = entry
    outname = f"out{comps}"
    if outname not in ctx.fields:
        ctx.add_field(outname, comps, 1, 0.0)
    ctx.fill(outname, 0.0)
    ops = [o if o in spec["fields"] else float(spec["consts"][o]) for o in operands]
    ctx.interact(name, ops, outname, kernel=kw)
    return ctx.download(outname)
