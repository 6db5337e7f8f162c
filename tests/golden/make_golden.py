"""Regenerate the golden fixtures in tests/golden/ from the reference itself.

Run in the build container (needs oracle/_ref/libnauticle_ref.so, i.e. the
reference sources compiled unmodified against oracle/shim/):

    make -C oracle && python tests/golden/make_golden.py

Every output below comes from the reference's own code path — ParticleSystem
cell tables / for_each_neighbor, the operator evaluators through the SFL
parser (or, for the two laws the reference lacks — cubic spline, linear
spring-dashpot — rules passed to its interact()), and Case::solve_step for the
dam-break deck. The fixtures are what tests/test_golden.py checks the C port
and the CUDA path against on machines without /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import ref  # noqa: E402
from paper_1710_08259_b200 import scenes  # noqa: E402
import cases  # noqa: E402


def pack_spec(prefix, spec, out):
    meta = {k: spec[k] for k in ("dim", "min_cells", "max_cells", "cell_size", "kinds")}
    meta = json.loads(json.dumps(meta, default=int))
    meta["consts"] = spec["consts"]
    meta["fields"] = sorted(spec["fields"])
    out[prefix + "meta"] = np.array(json.dumps(meta))
    out[prefix + "pos"] = spec["pos"]
    for k, v in spec["fields"].items():
        out[prefix + "f_" + k] = np.asarray(v)


def random_cases(out, count=16, seed=20261020):
    rng = np.random.default_rng(seed)
    specs = []
    # edge layouts first: single particle, empty, 1- and 2-cell periodic axes,
    # all-symmetric corner cells, then random mixes
    specs.append(cases.random_spec(rng, dim=3, n=1, kinds=[1, 1, 1], cells=[1, 1, 1]))
    specs.append(cases.random_spec(rng, dim=2, n=0, kinds=[0, 2], cells=[3, 2]))
    specs.append(cases.random_spec(rng, dim=3, n=60, kinds=[0, 0, 0], cells=[1, 2, 3]))
    specs.append(cases.random_spec(rng, dim=2, n=80, kinds=[1, 1], cells=[2, 2]))
    specs.append(cases.random_spec(rng, dim=1, n=40, kinds=[0], cells=[2]))
    while len(specs) < count:
        specs.append(cases.random_spec(rng))
    for idx, spec in enumerate(specs):
        p = f"c{idx}_"
        pack_spec(p, spec, out)
        rc = cases.ref_case(spec)
        nc = int(np.prod(spec["max_cells"]))
        cell_of, start, cnt, srt = rc.cell_tables(nc)
        out[p + "cell_of"], out[p + "cell_start"], out[p + "cell_count"], out[p + "sorted"] = \
            cell_of, start, cnt, srt
        out[p + "counts"] = rc.neighbor_counts(spec["consts"]["R"])
        for k, entry in enumerate(cases.op_list(spec["dim"])):
            try:
                out[p + f"op{k}"] = cases.ref_eval(spec, rc, entry)
            except ref.RefError as e:  # e.g. coincident gravity bodies
                out[p + f"op{k}_error"] = np.array(str(e))
    out["n_random_cases"] = np.array(len(specs))


def dam_break_case(out, steps=10):
    sc = scenes.dam_break(2, dx=0.1, fluid=(1.0, 1.0), tank=(2.0, 1.6))
    prm = sc.params
    rc = ref.RefCase(2, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds, sc.pos)
    for k in ("rho", "p", "v", "vdot", "mask"):
        rc.field(k, sc.fields[k])
    rc.constant("one", 1.0).constant("mass", prm["mass"]).constant("R", prm["radius"])
    rc.constant("B", prm["B"]).constant("rho0", prm["rho0"]).constant("gam", prm["gamma"])
    rc.constant("visc", prm["visc"]).constant("g", prm["g"]).variable("dt", prm["dt"])
    for name, text in scenes.wcsph_equations(sc):
        rc.equation(name, text)
    out["dam_meta"] = np.array(json.dumps({"dx": 0.1, "fluid": [1.0, 1.0], "tank": [2.0, 1.6],
                                           "steps": steps}))
    for s in range(1, steps + 1):
        rc.solve_step(1)
        if s in (1, steps):
            for k in ("r", "rho", "p", "v", "vdot"):
                out[f"dam_s{s}_{k}"] = rc.get(k)
            out[f"dam_s{s}_active"] = rc.active()


def microbench_case(out, n=4096):
    sc = scenes.sph_microbench(n=n)
    prm = sc.params
    rc = ref.RefCase(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds, sc.pos)
    rc.field("A", sc.fields["A"]).constant("one", 1.0).constant("m", prm["mass"])
    rc.constant("R", prm["radius"])
    out["mb_n"] = np.array(n)
    nc = int(np.prod(sc.max_cells))
    cell_of, start, cnt, srt = rc.cell_tables(nc)
    out["mb_cell_start"], out["mb_sorted"] = start, srt
    out["mb_counts"] = rc.neighbor_counts(prm["radius"])
    rho = rc.eval("sph_S(one,m,one,Wp53220,R)", 1)
    rc.field("rho", rho)
    out["mb_rho_w"] = rho
    out["mb_G_w"] = rc.eval("sph_G11(A,m,rho,Wp53220,R)", 3)
    out["mb_L_w"] = rc.eval("sph_L0(A,m,rho,Wp53220,R)", 1)
    out["mb_rho_c"] = rc.eval_law("sph_S", ["one", "m", "one", "R"], 1, kdim=3)
    out["mb_G_c"] = rc.eval_law("sph_G11", ["A", "m", "rho", "R"], 3, kdim=3)
    out["mb_L_c"] = rc.eval_law("sph_L0", ["A", "m", "rho", "R"], 1, kdim=3)


def main():
    assert ref.available(), "build oracle/_ref first: make -C oracle"
    out = {}
    random_cases(out)
    np.savez_compressed(os.path.join(HERE, "random_cases.npz"), **out)
    out = {}
    dam_break_case(out)
    np.savez_compressed(os.path.join(HERE, "dam_break_2d_small.npz"), **out)
    out = {}
    microbench_case(out)
    np.savez_compressed(os.path.join(HERE, "microbench_small.npz"), **out)
    draws = ref.uniform_draws(1, 257, 5)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), seed=1, draws=draws)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
