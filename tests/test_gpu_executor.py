"""GPU tests of the device equation executor (nau_case_*, csrc/executor.cpp), the
§8(b) "Caller": the reference's own shipped decks solved on the GPU against the
reference's Case::solve_step (tests/golden/decks.npz, written by
tests/golden/make_deck_golden.py from oracle/_ref, the unmodified reference sources).

* dam_break_2d, hot_start_demo (continuity sph_D00, two equations writing vdot,
  symmetric walls), sampling_1k (sph_S over a periodic box): EXACT mode is BITWISE
  equal to the reference for 10 steps (no libm transcendental on the path).
* cahn_hilliard_patch (c^3 through the device pow, an fmax reduction feeding the
  variable dt, periodic), particle_damper (fsum(dem_boundary_force) feeding a
  variable, Hertz dem_l with libm pow), sfm_agent (exp): within 1e-10 after 1 step and
  1e-6 after 10 (north_star), variables included.
* FAST mode: every deck within the same tolerances.
* Assembly errors of the reference's malformed decks and solve-time errors (shapes,
  NaN audit, variable LHS) with the reference's messages and error kinds.
"""
import json
import os

import numpy as np
import pytest

from paper_1710_08259_b200 import nau

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "decks.npz")
Z = np.load(GOLD)
INDEX = json.loads(str(Z["index"]))
BITWISE = {"dam_break_2d", "hot_start_demo", "sampling_1k"}
TOL = {1: 1e-10, 10: 1e-6}


def rel_err(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    scale = max(np.abs(b).max(initial=0.0), 1e-300)
    return float(np.abs(a - b).max(initial=0.0) / scale)


def build(prefix, meta, fast=False, fields_from=None):
    """Context + executor mirroring the assembled reference case (what a reference-side
    binding does with Case::workspace and Case::equations)."""
    d = meta["domain"]
    ctx = nau.Context(0)
    ctx.set_mode(fast)
    ctx.set_domain(d["dim"], d["min_cells"], d["max_cells"], d["cell_size"], d["kinds"])
    get = fields_from or (lambda f: Z[f"{prefix}_s0_{f}"])
    ctx.set_particles(get("r"))
    for fname, shape in meta["fields"]:
        if fname != "r":
            ctx.add_field(fname, shape[0], shape[1], get(fname))
    if "seed" in meta:
        ctx.set_random_state(meta["seed"], Z[f"{prefix}_s0_rand"])
    cs = nau.Case(ctx)
    for name, v in meta["constants"]:
        cs.constant(name, np.array(v))
    for name, v in meta["variables"]:
        cs.variable(name, np.array(v))
    return ctx, cs


@pytest.mark.parametrize("fast", [False, True])
@pytest.mark.parametrize("deck", INDEX["decks"])
def test_reference_deck_vs_case_solve_step(deck, fast):
    meta = json.loads(str(Z[f"{deck}_meta"]))
    ctx, cs = build(deck, meta, fast)
    try:
        for name, text in meta["equations"]:
            cs.equation(name, text)
        last = max(meta["steps"])
        for s in range(1, last + 1):
            cs.solve_step()
            if s not in meta["steps"]:
                continue
            np.testing.assert_array_equal(ctx.active(), Z[f"{deck}_s{s}_active"])
            exact = deck in BITWISE and not fast
            for fname, _ in meta["fields"]:
                got, exp = ctx.download(fname) if fname != "r" else ctx.download("r"), \
                    Z[f"{deck}_s{s}_{fname}"]
                if exact:
                    np.testing.assert_array_equal(got, exp, err_msg=f"step {s} field {fname}")
                else:
                    assert rel_err(got, exp) <= TOL[s], (s, fname, rel_err(got, exp))
            for vname, v in json.loads(str(Z[f"{deck}_s{s}_vars"])):
                got, exp = cs.get_variable(vname), np.array(v)
                if exact:
                    np.testing.assert_array_equal(got, exp, err_msg=f"step {s} variable {vname}")
                else:
                    assert rel_err(got, exp) <= TOL[s], (s, vname, got, exp)
    finally:
        ctx.close()


@pytest.mark.parametrize("case", INDEX["errors"])
def test_assembly_errors_like_the_reference(case):
    """The reference's malformed decks (tests/decks/malformed): the equation is rejected
    when added, with the reference's assembly message (assemble.cpp:171-196,
    sfl/parser.cpp)."""
    meta = json.loads(str(Z[f"err_{case}_meta"]))
    ctx, cs = build(f"err_{case}", meta,
                    fields_from=lambda f: Z[f"err_{case}_r"] if f == "r" else Z[f"err_{case}_f_{f}"])
    try:
        with pytest.raises(nau.NauError) as ei:
            for name, text in meta["equations"]:
                cs.equation(name, text)
        assert str(ei.value).endswith(meta["message"]), (str(ei.value), meta["message"])
    finally:
        ctx.close()


@pytest.mark.parametrize("case", INDEX["runtime_errors"])
def test_solve_errors_like_the_reference(case):
    """Equations that assemble but fail when solved (appended to dam_break_2d): the
    reference's message, prefixed "equation '<name>': ", and kind (NaN audit -> Nan)."""
    spec = json.loads(str(Z[f"rt_{case}"]))
    meta = json.loads(str(Z["dam_break_2d_meta"]))
    ctx, cs = build("dam_break_2d", meta)
    try:
        for name, text in meta["equations"] + [[case, spec["text"]]]:
            cs.equation(name, text)
        with pytest.raises(nau.NauError) as ei:
            cs.solve_step()
        assert str(ei.value).endswith(spec["message"]), (str(ei.value), spec["message"])
        want = 2 if "non-finite" in spec["message"] else 1  # NAU_ERR_NAN / NAU_ERR_RUNTIME
        assert ei.value.status == want
    finally:
        ctx.close()


def test_executor_equals_the_fused_deck():
    """The BASELINE WCSPH deck as equations through the executor equals nau_wcsph_step's
    fused passes (EXACT mode: both bitwise to the reference), over 3 steps."""
    from paper_1710_08259_b200 import scenes
    sc = scenes.dam_break(2, dx=0.05, fluid=(0.5, 1.0), tank=(1.5, 1.2))
    prm = sc.params
    out = []
    for use_case in (False, True):
        ctx = nau.Context(0)
        try:
            ctx.set_domain(2, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
            ctx.set_particles(sc.pos)
            for k in ("rho", "p", "v", "vdot", "mask"):
                v = np.asarray(sc.fields[k]).reshape(-1, sc.n)
                ctx.add_field(k, v.shape[0], 1, v)
            ctx.boundary_shift()
            if use_case:
                cs = nau.Case(ctx)
                cs.constant("one", 1.0).constant("mass", prm["mass"]).constant("R", prm["radius"])
                cs.constant("B", prm["B"]).constant("rho0", prm["rho0"]).constant("gam", prm["gamma"])
                cs.constant("visc", prm["visc"]).constant("g", np.array(prm["g"]))
                cs.variable("dt", prm["dt"])
                for name, text in scenes.wcsph_equations(sc):
                    cs.equation(name, text)
                for _ in range(3):
                    cs.solve_step()
            else:
                p = nau.WcsphParams()
                p.kernel_family, p.kernel_dim = nau.K_WENDLAND, 2
                p.mass, p.radius, p.rho0, p.B = prm["mass"], prm["radius"], prm["rho0"], prm["B"]
                p.gamma, p.visc, p.dt = prm["gamma"], prm["visc"], prm["dt"]
                p.g[0], p.g[1] = prm["g"]
                f = ctx.fields
                p.f_rho, p.f_p, p.f_v, p.f_vdot, p.f_mask = (f["rho"].id, f["p"].id, f["v"].id,
                                                             f["vdot"].id, f["mask"].id)
                for _ in range(3):
                    ctx.wcsph_step(p)
            out.append({k: ctx.download(k) for k in ("r", "rho", "v", "vdot")})
        finally:
            ctx.close()
    for k in out[0]:
        assert rel_err(out[1][k], out[0][k]) <= 1e-12, k  # Tait pow: device vs host libm


@pytest.mark.parametrize("deck", ["cahn_hilliard_patch", "particle_damper"])
def test_reductions_through_a_communicator(deck):
    """With a communicator attached (nau_comm_init), every reduction of the executor goes
    through ncclAllReduce (nau_allreduce: the §8(e) reduction over slab ranks): on a
    1-rank communicator the decks' fmax -> dt and fsum -> F results equal the run without
    one bitwise."""
    meta = json.loads(str(Z[f"{deck}_meta"]))
    runs = []
    for comm in (False, True):
        ctx, cs = build(deck, meta)
        try:
            if comm:
                ctx.comm_init(nau.Context.comm_unique_id(), 1, 0)
            for name, text in meta["equations"]:
                cs.equation(name, text)
            for _ in range(3):
                cs.solve_step()
            runs.append({vn: cs.get_variable(vn) for vn, _ in meta["variables"]})
        finally:
            ctx.close()
    for vn in runs[0]:
        np.testing.assert_array_equal(runs[1][vn], runs[0][vn], err_msg=vn)


def test_allreduce_ops_on_one_rank():
    ctx = nau.Context(0)
    try:
        ctx.set_domain(1, [0], [1], [1.0], [nau.CUTOFF])
        ctx.set_particles(np.array([[0.5]]))
        L = ctx.L
        v = np.array([1.5, -2.0, 3.0])
        assert L.nau_comm_size(ctx.h) == 1
        assert L.nau_allreduce(ctx.h, v.ctypes.data_as(nau.C.c_void_p), 3, 0) == 0  # no comm
        ctx.comm_init(nau.Context.comm_unique_id(), 1, 0)
        for op in (0, 1, 2):
            w = v.copy()
            assert L.nau_allreduce(ctx.h, w.ctypes.data_as(nau.C.c_void_p), 3, op) == 0
            np.testing.assert_array_equal(w, v)
        assert L.nau_allreduce(ctx.h, v.ctypes.data_as(nau.C.c_void_p), 3, 7) != 0
    finally:
        ctx.close()
