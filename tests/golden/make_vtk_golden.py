"""Regenerate the result-frame fixtures (tests/golden/frame_*.vtk) from the reference.

    make -C oracle && python tests/golden/make_vtk_golden.py

A small 3D case (periodic / symmetric / cut-off axes, one particle past the
cut-off wall, hence inactive) with a scalar, a 3-vector, a 2-vector and a 3x3
field, a vector and a scalar constant, a variable and one equation that draws
rand(0,1) is stepped once through Case::solve_step; the reference's own
make_frame + write_vtk (io/vtk.cpp:193-304) then writes it as ASCII and BINARY
legacy VTK. frame_case.npz holds the inputs the GPU test rebuilds the state from.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402

SEED, N = 11, 40


def main():
    assert ref.available(), "build oracle/_ref first: make -C oracle"
    rng = np.random.default_rng(SEED)
    pos = rng.uniform(0.0, 1.0, (3, N))
    pos[2, 5] = 1.3  # past the cut-off wall: deactivated at assembly
    kinds = [0, 1, 2]
    rc = ref.RefCase(3, [0, 0, 0], [2, 2, 2], [0.5, 0.5, 0.5], kinds, pos, seed=SEED)
    fields = {"rho": rng.uniform(900, 1100, (1, N)), "v": rng.normal(size=(3, N)),
              "w2": rng.normal(size=(2, N)), "S": rng.normal(size=(9, N))}
    shapes = {"rho": (1, 1), "v": (3, 1), "w2": (2, 1), "S": (3, 3)}
    for k, v in fields.items():
        rc.field(k, v, rows=shapes[k][0], cols=shapes[k][1])
    rc.constant("g", np.array([0.0, 0.0, -9.81])).constant("k", 0.1)
    rc.variable("dt", 1e-3)
    rc.equation("rhoeq", "rho=rho+k*rand(0,1)")
    rc.solve_step()
    rc.write_vtk(os.path.join(HERE, "frame_ascii.vtk"), False, 7, 0.125, 2.5)
    rc.write_vtk(os.path.join(HERE, "frame_binary.vtk"), True, 7, 0.125, 2.5)
    out = {"pos": rc.get("r"), "active": rc.active(), "seed": SEED,
           "kinds": np.array(kinds), "field_order": np.array(list(fields))}
    for k in fields:
        out["f_" + k] = rc.get(k)
        out["shape_" + k] = np.array(shapes[k])
    np.savez_compressed(os.path.join(HERE, "frame_case.npz"), **out)
    print("frame fixtures written to", HERE)


if __name__ == "__main__":
    main()
