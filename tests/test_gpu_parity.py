"""GPU parity tests: the CUDA path through the C-ABI vs the oracle.

Integer data (cell ids, cell tables, sorted order, neighbour counts) must be
bit-exact. The SPH operators and the linear spring-dashpot law are compiled
without FMA contraction and sum in the reference's candidate order, so they
are checked bitwise too. Paths through a libm transcendental (Hertz pow,
gravity's r^1.5, the Tait EOS pow) use BASELINE's fp64 tolerance: 1e-10
relative for one step, 1e-6 relative after 10 steps (north_star).
"""
import json
import os

import numpy as np
import pytest

import cases
import deck_oracle
from oracle import port
from paper_1710_08259_b200 import nau, scenes

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL_STEP = 1e-10
TOL_10 = 1e-6
TRANSCENDENTAL = {"dem_l", "dem_boundary_force", "nbody_gravity", "sfm"}  # libm pow/exp


def rel_err(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    scale = max(np.abs(b).max(initial=0.0), 1e-300)
    return float(np.abs(a - b).max(initial=0.0) / scale)


@pytest.fixture(scope="module")
def ctx():
    c = nau.Context(0)
    yield c
    c.close()


def unpack_spec(z, p):
    meta = json.loads(str(z[p + "meta"]))
    spec = {k: meta[k] for k in ("dim", "min_cells", "max_cells", "cell_size", "kinds")}
    spec["consts"] = meta["consts"]
    spec["pos"] = z[p + "pos"]
    spec["fields"] = {k: z[p + "f_" + k] for k in meta["fields"]}
    return spec


def check_against(spec, ctx, expect_tables, expect_counts, expect_ops):
    cases.gpu_context(spec, ctx)
    tables = ctx.cell_tables()
    for got, exp, name in zip(tables, expect_tables, ("cell_of", "start", "count", "sorted")):
        np.testing.assert_array_equal(got, exp, err_msg=name)
    np.testing.assert_array_equal(ctx.neighbor_counts(spec["consts"]["R"]), expect_counts)
    for entry, exp in zip(cases.op_list(spec["dim"]), expect_ops):
        if exp is None:
            continue
        got = cases.gpu_eval(spec, ctx, entry)
        if entry[0] in TRANSCENDENTAL:
            assert rel_err(got, exp) <= TOL_STEP, entry[0]
        else:
            np.testing.assert_array_equal(got, exp, err_msg=f"{entry[0]} {entry[2]}")


@pytest.mark.parametrize("idx", range(16))
def test_golden_random_cases(ctx, idx):
    z = np.load(os.path.join(GOLD, "random_cases.npz"))
    if idx >= int(z["n_random_cases"]):
        pytest.skip()
    p = f"c{idx}_"
    spec = unpack_spec(z, p)
    ops = [None if p + f"op{k}_error" in z else z[p + f"op{k}"]
           for k in range(len(cases.op_list(spec["dim"])))]
    check_against(spec, ctx, [z[p + s] for s in ("cell_of", "cell_start", "cell_count", "sorted")],
                  z[p + "counts"], ops)


@pytest.mark.parametrize("seed", range(8))
def test_live_random_cases_vs_port(ctx, seed):
    rng = np.random.default_rng(77 + seed)
    spec = cases.random_spec(rng, n=int(rng.integers(500, 3000)), cells=None)
    ps = cases.port_system(spec)
    ops = [cases.port_eval(spec, ps, e) for e in cases.op_list(spec["dim"])]
    check_against(spec, ctx, ps.tables, ps.neighbor_counts(spec["consts"]["R"]), ops)


def test_edge_layouts(ctx):
    rng = np.random.default_rng(5)
    # everything in one cell (large ppc), periodic 1-cell axes visited three times
    spec = cases.random_spec(rng, dim=3, n=1500, kinds=[0, 0, 0], cells=[1, 1, 1])
    ps = cases.port_system(spec)
    ops = [cases.port_eval(spec, ps, e) for e in cases.op_list(3)]
    check_against(spec, ctx, ps.tables, ps.neighbor_counts(spec["consts"]["R"]), ops)
    # particles exactly on cell faces and on the periodic seam
    spec = cases.random_spec(rng, dim=2, n=400, kinds=[0, 1], cells=[4, 3])
    pos = spec["pos"]
    pos[0, :100] = np.round(pos[0, :100] / 0.3) * 0.3
    pos[0, 100:110] = np.nextafter(1.2, 0.0)
    pos[1, 110:130] = 0.0
    ps = cases.port_system(spec)
    ops = [cases.port_eval(spec, ps, e) for e in cases.op_list(2)]
    check_against(spec, ctx, ps.tables, ps.neighbor_counts(spec["consts"]["R"]), ops)


def test_empty_and_single(ctx):
    rng = np.random.default_rng(6)
    spec = cases.random_spec(rng, dim=2, n=0, kinds=[0, 2], cells=[3, 2])
    cases.gpu_context(spec, ctx)
    cell_of, start, count, srt = ctx.cell_tables()
    assert count.sum() == 0 and len(srt) == 0 and (start == 0).all()
    spec = cases.random_spec(rng, dim=3, n=1, kinds=[1, 1, 1], cells=[1, 1, 1])
    ps = cases.port_system(spec)
    ops = [cases.port_eval(spec, ps, e) for e in cases.op_list(3)]
    check_against(spec, ctx, ps.tables, ps.neighbor_counts(spec["consts"]["R"]), ops)


def test_cutoff_leavers_are_deactivated_and_frozen(ctx):
    rng = np.random.default_rng(8)
    spec = cases.random_spec(rng, dim=2, n=600, kinds=[2, 0], cells=[5, 4])
    spec["pos"][0, :37] = -0.05   # outside the cut-off face: deactivated by the shift
    spec["pos"][0, 37:50] = 1.52  # beyond hi = 1.5
    ps = cases.port_system(spec)
    assert ps.active.sum() == 550
    cases.gpu_context(spec, ctx)
    np.testing.assert_array_equal(ctx.active(), ps.active)
    ops = [cases.port_eval(spec, ps, e) for e in cases.op_list(2)]
    check_against(spec, ctx, ps.tables, ps.neighbor_counts(spec["consts"]["R"]), ops)


def test_errors_surface_like_the_reference(ctx):
    rng = np.random.default_rng(9)
    spec = cases.random_spec(rng, dim=2, n=300, kinds=[0, 0], cells=[4, 4])
    spec["fields"]["rho"][0, 17] = 0.0
    cases.gpu_context(spec, ctx)
    ctx.add_field("o", 2, 1, 0.0)
    ctx.interact("sph_G11", ["A", 0.5, "rho", 0.3], "o", kernel="Wp52220")
    with pytest.raises(nau.NauError) as e:  # interactions.cpp:92-94 zero density
        ctx.sync()
    assert e.value.status == 1 and "zero density" in e.value.message
    ctx.interact("sph_S", ["A", 0.5, "rho", -1.0], "o1" if "o1" in ctx.fields else
                 ctx.add_field("o1", 1, 1, 0.0), kernel="Wp52220")
    with pytest.raises(nau.NauError) as e:  # sph_context radius check
        ctx.sync()
    assert "radius" in e.value.message
    with pytest.raises(nau.NauError):  # D00 needs a vector operand
        ctx.interact("sph_D00", ["A", 0.5, "rho", 0.3], "o1", kernel="Wp52220")
    nan = spec["fields"]["A"].copy()
    nan[0, 5] = np.nan
    ctx.add_field("An", 1, 1, nan)
    ctx.interact("sph_L0", ["An", 0.5, 1000.0, 0.3], "o1", kernel="Wp52220")
    with pytest.raises(nau.NauError) as e:  # case.cpp:46-53 NaN audit
        ctx.sync()
    assert e.value.status == 2
    ctx.sync()  # error word cleared


def _sfm_ctx(pos, vel, tau=0.5, v0=1.3):
    """The reference's sfm KAT deck (test_interactions.cpp:408-420): 8 x 8 cut-off
    cells of 1 m, A = 2000, B = 0.08, k = 1.2e5, R = 0.25, c = 0, m = 70."""
    c = nau.Context(0)
    c.set_domain(2, [0, 0], [8, 8], [1.0, 1.0], [nau.CUTOFF, nau.CUTOFF])
    n = len(pos)
    c.set_particles(np.array(pos, dtype=np.float64).T.copy())
    c.add_field("v", 2, 1, np.array(vel, dtype=np.float64).T.copy())
    c.add_field("rdes", 2, 1, np.tile([[1000.0], [4.0]], (1, n)))
    c.add_field("a", 2, 1, 0.0)
    return c, ["v", v0, "rdes", 0.25, 2000.0, 0.08, 1.2e5, 0.0, 70.0, tau]


def test_sfm_reference_kats():
    """test_interactions.cpp:408-445 through the C-ABI: a relaxed agent feels no
    force, a resting one accelerates at v0/tau, an overlapping pair is symmetric
    and matches the hand formula."""
    v0, tau = 1.3, 0.5
    c, ops = _sfm_ctx([(4, 4)], [(v0, 0)])
    c.interact("sfm", ops, "a")
    assert np.linalg.norm(c.download("a")[:, 0]) <= 1e-9
    c.close()
    c, ops = _sfm_ctx([(4, 4)], [(0, 0)])
    c.interact("sfm", ops, "a")
    a = c.download("a")[:, 0]
    assert abs(a[0] - v0 / tau) <= 1e-6 * v0 / tau and abs(a[1]) <= 1e-5
    c.close()
    c, ops = _sfm_ctx([(4.0, 4.0), (4.3, 4.0)], [(0, 0), (0, 0)])
    ops[1] = 0.0
    c.interact("sfm", ops, "a")
    a = c.download("a")
    assert np.linalg.norm(a[:, 0] + a[:, 1]) <= 1e-12 * np.linalg.norm(a[:, 0])
    d, rij = 0.3, 0.5
    f = 2000.0 * np.exp((rij - d) / 0.08) + 1.2e5 * (rij - d)
    assert abs(a[0, 0] - (-f / 70.0)) <= 1e-12 * f / 70.0
    c.close()


def test_sfm_errors_and_warnings(ctx):
    """sfm's own checks (interactions.cpp:228-229; the lowest offending index),
    the Tensor shape messages of its operand algebra, and one warning per agent
    already at its desired position."""
    rng = np.random.default_rng(4)
    spec = cases.random_spec(rng, dim=2, n=200, kinds=[2, 2], cells=[3, 3])
    cases.gpu_context(spec, ctx)
    ctx.add_field("o2", 2, 1, 0.0)
    base = ["V", 1.3, "V", "Rp", 2.0, 0.08, 120.0, 0.05, "M", 0.5]
    for slot, msg in ((9, "relaxation time"), (8, "mass")):
        bad = list(base)
        bad[slot] = 0.0
        ctx.interact("sfm", bad, "o2")
        with pytest.raises(nau.NauError) as e:
            ctx.sync()
        assert e.value.status == 1 and f"sfm: {msg} must be positive" in e.value.message
    m = spec["fields"]["M"].copy()
    m[0, [37, 11, 90]] = -1.0
    ctx.add_field("Mbad", 1, 1, m)
    bad = list(base)
    bad[8] = "Mbad"
    ctx.interact("sfm", bad, "o2")
    with pytest.raises(nau.NauError) as e:
        ctx.sync()
    assert e.value.particle == 11
    for slot, text in ((2, "operator '-': incompatible shapes 1x1 and 2x1"),
                       (0, "operator '-': incompatible shapes 2x1 and 1x1"),
                       (4, "expected a scalar, got a 2x1 tensor")):
        bad = list(base)
        bad[slot] = "A" if slot != 4 else "V"
        with pytest.raises(nau.NauError) as e:
            ctx.interact("sfm", bad, "o2")
        assert text in e.value.message, e.value.message
    ctx.add_field("rhere", 2, 1, ctx.download("r"))
    w0 = ctx.warning_count
    at_goal = list(base)
    at_goal[2] = "rhere"
    ctx.interact("sfm", at_goal, "o2")
    ctx.sync()
    assert ctx.warning_count - w0 == 200
    ps = cases.port_system(spec)
    from oracle import port
    ops = [cases.port_operand(spec, o) if isinstance(o, str) and o != "rhere" else o
           for o in at_goal]
    ops[2] = ps.pos
    want = ps.interact(port.SFM, ops, (2, 1))
    assert rel_err(ctx.download("o2"), want) <= TOL_STEP


def test_microbench_golden(ctx):
    z = np.load(os.path.join(GOLD, "microbench_small.npz"))
    sc = scenes.sph_microbench(n=int(z["mb_n"]))
    prm = sc.params
    ctx.set_domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
    ctx.set_particles(sc.pos)
    ctx.add_field("A", 1, 1, sc.fields["A"])
    ctx.add_field("rho", 1, 1, 0.0)
    ctx.add_field("G", 3, 1, 0.0)
    ctx.add_field("L", 1, 1, 0.0)
    ctx.boundary_shift()
    _, start, _, srt = ctx.cell_tables()
    np.testing.assert_array_equal(start, z["mb_cell_start"])
    np.testing.assert_array_equal(srt, z["mb_sorted"])
    np.testing.assert_array_equal(ctx.neighbor_counts(prm["radius"]), z["mb_counts"])
    ctx.add_field("rho_w", 1, 1, z["mb_rho_w"])
    for kw, sfx in (("Wp53220", "w"), ("Wc33220", "c")):
        ctx.interact("sph_S", [1.0, prm["mass"], 1.0, prm["radius"]], "rho", kernel=kw)
        ctx.interact("sph_G11", ["A", prm["mass"], "rho_w", prm["radius"]], "G", kernel=kw)
        ctx.interact("sph_L0", ["A", prm["mass"], "rho_w", prm["radius"]], "L", kernel=kw)
        np.testing.assert_array_equal(ctx.download("rho"), z["mb_rho_" + sfx])
        np.testing.assert_array_equal(ctx.download("G"), z["mb_G_" + sfx])
        np.testing.assert_array_equal(ctx.download("L"), z["mb_L_" + sfx])


def test_microbench_full_size(ctx):
    """BASELINE cfg1 at its full N = 1,048,576: bit-exact tables and counts, bitwise density."""
    sc = scenes.sph_microbench()
    prm = sc.params
    ctx.set_domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
    ctx.set_particles(sc.pos)
    ctx.add_field("rho", 1, 1, 0.0)
    ctx.boundary_shift()
    dom = port.Domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
    ps = port.ParticleSystem(dom, sc.pos)
    ps.boundary_shift()
    ps.build_cells()
    for got, exp in zip(ctx.cell_tables(), ps.tables):
        np.testing.assert_array_equal(got, exp)
    counts = ctx.neighbor_counts(prm["radius"])
    np.testing.assert_array_equal(counts, ps.neighbor_counts(prm["radius"]))
    assert abs(counts.mean() - 51.0) < 0.5  # 50 expected neighbours + self
    ctx.interact("sph_S", [1.0, prm["mass"], 1.0, prm["radius"]], "rho", kernel="Wc33220")
    rho = ctx.download("rho")
    np.testing.assert_array_equal(
        rho, ps.interact(port.SPH_S, [1.0, prm["mass"], 1.0, prm["radius"]], (1, 1),
                         kfamily=port.K_CUBIC))


def _gpu_dam(ctx, sc):
    prm = sc.params
    ctx.set_domain(sc.dim, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
    ctx.set_particles(sc.pos)
    for k in ("rho", "p", "v", "vdot", "mask"):
        v = np.asarray(sc.fields[k]).reshape(-1, sc.n)
        ctx.add_field(k, v.shape[0], 1, v)
    ctx.boundary_shift()
    p = nau.WcsphParams()
    p.kernel_family, p.kernel_dim = nau.K_WENDLAND, sc.dim
    p.mass, p.radius, p.rho0, p.B = prm["mass"], prm["radius"], prm["rho0"], prm["B"]
    p.gamma, p.visc, p.dt = prm["gamma"], prm["visc"], prm["dt"]
    for a in range(sc.dim):
        p.g[a] = prm["g"][a]
    f = ctx.fields
    p.f_rho, p.f_p, p.f_v, p.f_vdot, p.f_mask = (f["rho"].id, f["p"].id, f["v"].id,
                                                 f["vdot"].id, f["mask"].id)
    return p


def test_dam_break_small_vs_reference_golden(ctx):
    z = np.load(os.path.join(GOLD, "dam_break_2d_small.npz"))
    meta = json.loads(str(z["dam_meta"]))
    sc = scenes.dam_break(2, dx=meta["dx"], fluid=tuple(meta["fluid"]), tank=tuple(meta["tank"]))
    p = _gpu_dam(ctx, sc)
    for s in range(1, meta["steps"] + 1):
        ctx.wcsph_step(p)
        if s in (1, meta["steps"]):
            tol = TOL_STEP if s == 1 else TOL_10
            assert rel_err(ctx.download("r"), z[f"dam_s{s}_r"]) <= tol
            for k in ("rho", "p", "v", "vdot"):
                assert rel_err(ctx.download(k), z[f"dam_s{s}_{k}"]) <= tol, (s, k)
            np.testing.assert_array_equal(ctx.active(), z[f"dam_s{s}_active"])


def test_dam_break_cfg0_full_vs_port_10_steps(ctx):
    """BASELINE cfg0 (23,018 particles): 1 step within 1e-10, 10 steps within 1e-6,
    mass exactly conserved (no particle lost), momentum consistent."""
    sc = scenes.dam_break(2)
    prm = sc.params
    p = _gpu_dam(ctx, sc)
    ps, st = deck_oracle.make_system(sc)
    for s in range(1, 11):
        ctx.wcsph_step(p)
        deck_oracle.step(ps, st, prm)
        if s in (1, 10):
            tol = TOL_STEP if s == 1 else TOL_10
            assert rel_err(ctx.download("r"), ps.pos) <= tol
            for k in ("rho", "p", "v"):
                assert rel_err(ctx.download(k), st[k]) <= tol, (s, k)
    act = ctx.active()
    np.testing.assert_array_equal(act, ps.active)
    assert act.sum() * prm["mass"] == sc.n * prm["mass"]  # mass conserved exactly
    mom_g = (ctx.download("v") * prm["mass"]).sum(axis=1)
    mom_o = (st["v"] * prm["mass"]).sum(axis=1)
    assert np.abs(mom_g - mom_o).max() <= 1e-8 * max(np.abs(mom_o).max(), 1e-30)


def test_euler_and_reduce(ctx):
    rng = np.random.default_rng(12)
    spec = cases.random_spec(rng, dim=3, n=2000, kinds=[0, 1, 2], cells=[3, 3, 3])
    cases.gpu_context(spec, ctx)
    ctx.add_field("V2", 3, 1, 0.0)
    ctx.euler("V", "V", 0.25, "V2")
    V = spec["fields"]["V"]
    np.testing.assert_array_equal(ctx.download("V2"), V + 0.25 * V)
    s = ctx.reduce("fsum", "A")
    assert abs(s[0] - spec["fields"]["A"].sum()) <= 1e-12 * spec["fields"]["A"].sum()
    assert ctx.reduce("fmax", "A")[0] == spec["fields"]["A"].max()
    nrm = np.sqrt((V * V).sum(axis=0))
    assert ctx.reduce("fmin", "V")[0] == pytest.approx(nrm.min(), rel=1e-15)


# ---------------------------------------------------------------- FAST mode ----
SPH_NAMES = {"sph_S", "sph_D00", "sph_G11", "sph_L0", "sph_A"}


@pytest.mark.parametrize("seed", range(6))
def test_fast_mode_matches_exact(ctx, seed):
    """FAST mode (warp per particle, FMA/rsqrt, tree sums) vs EXACT on the same inputs."""
    rng = np.random.default_rng(300 + seed)
    spec = cases.random_spec(rng, n=int(rng.integers(300, 3000)))
    cases.gpu_context(spec, ctx)
    for entry in cases.op_list(spec["dim"]):
        if entry[0] not in SPH_NAMES:
            continue
        ctx.set_mode(False)
        exact = cases.gpu_eval(spec, ctx, entry)
        ctx.set_mode(True)
        fast = cases.gpu_eval(spec, ctx, entry)
        ctx.set_mode(False)
        assert rel_err(fast, exact) <= 1e-12, (entry[0], entry[2], rel_err(fast, exact))


def test_fast_mode_microbench_full_size(ctx):
    sc = scenes.sph_microbench()
    prm = sc.params
    ctx.set_domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
    ctx.set_particles(sc.pos)
    ctx.add_field("A", 1, 1, sc.fields["A"])
    for f, r in (("rho", 1), ("G", 3), ("L", 1)):
        ctx.add_field(f, r, 1, 0.0)
    ctx.boundary_shift()
    out = {}
    for fast in (False, True):
        ctx.set_mode(fast)
        ctx.interact("sph_S", [1.0, prm["mass"], 1.0, prm["radius"]], "rho", kernel="Wc33220")
        ctx.interact("sph_G11", ["A", prm["mass"], "rho", prm["radius"]], "G", kernel="Wc33220")
        ctx.interact("sph_L0", ["A", prm["mass"], "rho", prm["radius"]], "L", kernel="Wc33220")
        out[fast] = {k: ctx.download(k) for k in ("rho", "G", "L")}
    ctx.set_mode(False)
    for k in ("rho", "G", "L"):
        assert rel_err(out[True][k], out[False][k]) <= TOL_STEP, k


@pytest.mark.parametrize("seed", range(6))
def test_fused_g11_l0_equals_two_calls(seed):
    """nau_interact_g11_l0 (one list walk for sph_G11 + sph_L0) = the two nau_interact
    calls bitwise, FAST and EXACT, incl. image/mirror domains, coincident-particle
    warnings and aliasing fall-backs."""
    rng = np.random.default_rng(900 + seed)
    spec = cases.random_spec(rng, dim=int(rng.integers(2, 4)), n=int(rng.integers(300, 3000)))
    if seed % 2:  # coincident distinct particles: sph_L0 warns, sph_G11 skips
        spec["pos"][:, 1] = spec["pos"][:, 0]
    dim = spec["dim"]
    m, R = float(spec["consts"]["m"]), float(spec["consts"]["R"])
    for kw in (f"Wp5{dim}220", f"Wc3{dim}220"):
        for fast in (True, False):
            for ops in (["A", m, "rho", R], ["A", "M", "rho", R]):
                res = []
                for fused in (False, True):
                    c = cases.gpu_context(spec)
                    c.set_mode(fast)
                    c.add_field("G", dim, 1, 0.0)
                    c.add_field("L", 1, 1, 0.0)
                    w0 = c.warning_count
                    if fused:
                        c.interact_g11_l0(ops, "G", "L", kernel=kw)
                    else:
                        c.interact("sph_G11", ops, "G", kernel=kw)
                        c.interact("sph_L0", ops, "L", kernel=kw)
                    c.sync()
                    res.append((c.download("G"), c.download("L"), c.warning_count - w0))
                    c.close()
                np.testing.assert_array_equal(res[1][0], res[0][0])
                np.testing.assert_array_equal(res[1][1], res[0][1])
                assert res[1][2] == res[0][2]
                if seed % 2:
                    assert res[0][2] > 0


def test_fused_g11_l0_microbench_full_size(ctx):
    """cfg1 at full size: the fused pass equals sph_G11 then sph_L0 bitwise (FAST)."""
    sc = scenes.sph_microbench()
    prm = sc.params
    ctx.set_domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
    ctx.set_particles(sc.pos)
    ctx.add_field("A", 1, 1, sc.fields["A"])
    for f, r in (("rho", 1), ("G", 3), ("L", 1)):
        ctx.add_field(f, r, 1, 0.0)
    ctx.boundary_shift()
    ctx.set_mode(True)
    ops = ["A", prm["mass"], "rho", prm["radius"]]
    ctx.interact("sph_S", [1.0, prm["mass"], 1.0, prm["radius"]], "rho", kernel="Wc33220")
    ctx.interact("sph_G11", ops, "G", kernel="Wc33220")
    ctx.interact("sph_L0", ops, "L", kernel="Wc33220")
    ref = ctx.download("G"), ctx.download("L")
    ctx.fill("G", 0.0)
    ctx.fill("L", 0.0)
    ctx.interact_g11_l0(ops, "G", "L", kernel="Wc33220")
    ctx.set_mode(False)
    np.testing.assert_array_equal(ctx.download("G"), ref[0])
    np.testing.assert_array_equal(ctx.download("L"), ref[1])


def test_fused_g11_l0_errors_like_two_calls():
    """rho_j == 0 / rho_i == 0: same error (message, particle) as the two calls; an
    output aliasing an operand takes the two-call path."""
    rng = np.random.default_rng(77)
    spec = cases.random_spec(rng, dim=3, n=800)
    spec["fields"]["rho"][0, 123] = 0.0
    msgs = []
    for fused in (False, True):
        c = cases.gpu_context(spec)
        c.set_mode(True)
        c.add_field("G", 3, 1, 0.0)
        c.add_field("L", 1, 1, 0.0)
        with pytest.raises(nau.NauError) as ei:
            if fused:
                c.interact_g11_l0(["A", 0.5, "rho", 0.3], "G", "L", kernel="Wp53220")
            else:
                c.interact("sph_G11", ["A", 0.5, "rho", 0.3], "G", kernel="Wp53220")
                c.interact("sph_L0", ["A", 0.5, "rho", 0.3], "L", kernel="Wp53220")
            c.sync()
        msgs.append(str(ei.value))
        if fused:  # the reference never evaluates the sph_L0 equation: L keeps its values
            assert not np.any(c.download("L"))
        c.close()
    assert msgs[0] == msgs[1] and msgs[0]
    spec["fields"]["rho"][0, 123] = 1000.0
    outs = []
    for fused in (False, True):
        c = cases.gpu_context(spec)
        c.set_mode(True)
        c.add_field("G", 3, 1, 0.0)
        if fused:
            c.interact_g11_l0(["A", 0.5, "rho", 0.3], "G", "A", kernel="Wp53220")
        else:
            c.interact("sph_G11", ["A", 0.5, "rho", 0.3], "G", kernel="Wp53220")
            c.interact("sph_L0", ["A", 0.5, "rho", 0.3], "A", kernel="Wp53220")
        outs.append((c.download("G"), c.download("A")))
        c.close()
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


def test_fast_mode_dam_break_vs_port(ctx):
    """cfg0 deck in FAST mode: 1 step within 1e-10, 10 steps within 1e-6 of the oracle."""
    sc = scenes.dam_break(2)
    prm = sc.params
    p = _gpu_dam(ctx, sc)
    ctx.set_mode(True)
    ps, st = deck_oracle.make_system(sc)
    for s in range(1, 11):
        ctx.wcsph_step(p)
        deck_oracle.step(ps, st, prm)
        if s in (1, 10):
            tol = TOL_STEP if s == 1 else TOL_10
            assert rel_err(ctx.download("r"), ps.pos) <= tol
            for k in ("rho", "p", "v"):
                assert rel_err(ctx.download(k), st[k]) <= tol, (s, k)
    ctx.set_mode(False)
    np.testing.assert_array_equal(ctx.active(), ps.active)


# ------------------------------------------------------- neighbour lists ----
def _run_deck(build, fast, lists, steps):
    c = nau.Context(0)
    try:
        p = build(c)
        c.set_mode(fast)
        c.set_neighbor_lists(lists)
        for _ in range(steps):
            c.wcsph_step(p)
        return {k: c.download(k) for k in ("r", "rho", "p", "v", "vdot")}, c.active()
    finally:
        c.close()


def _random_deck(n, seed, kind, radius, outside=0):
    """n random particles in the unit square, 4 x 4 cells of 0.25 (lists of up
    to ~n pi radius^2 entries: exercises the list capacity growth/fallback).
    `outside` particles are moved just past x = 1 (clamped into the last cell
    column of a symmetric axis: the fp16 list pre-filter must step aside)."""
    def build(c):
        rng = np.random.default_rng(seed)
        c.set_domain(2, [0, 0], [4, 4], [0.25, 0.25], [kind, kind])
        pos = rng.random((2, n))
        pos[0, :outside] = 1.0 + 0.02 * rng.random(outside)
        c.set_particles(pos)
        c.add_field("rho", 1, 1, 0.0)
        c.add_field("p", 1, 1, 0.0)
        c.add_field("v", 2, 1, 0.01 * rng.standard_normal((2, n)))
        c.add_field("vdot", 2, 1, 0.0)
        c.add_field("mask", 1, 1, 1.0)
        p = nau.WcsphParams()
        p.kernel_family, p.kernel_dim = nau.K_WENDLAND, 2
        p.mass, p.radius, p.rho0, p.B = 1.0 / n, radius, 1.0, 1.0
        p.gamma, p.visc, p.dt = 7.0, 0.1, 1e-4
        p.g[1] = -1.0
        f = c.fields
        p.f_rho, p.f_p, p.f_v, p.f_vdot, p.f_mask = (f["rho"].id, f["p"].id, f["v"].id,
                                                     f["vdot"].id, f["mask"].id)
        return p
    return build


@pytest.mark.parametrize("fast", [False, True])
def test_neighbor_lists_identical_to_sweep_dam3d(fast):
    """The per-step lists visit the sweep's candidates in the sweep's order: bitwise
    identical results with lists on and off (3D dam break, both modes)."""
    build = lambda c: _gpu_dam(c, scenes.dam_break(3, dx=0.02))
    off, act_off = _run_deck(build, fast, 0, 3)
    for mode in (1, 2):  # paired lists (FAST), per-particle lists
        on, act_on = _run_deck(build, fast, mode, 3)
        np.testing.assert_array_equal(act_on, act_off)
        for k in on:
            np.testing.assert_array_equal(on[k], off[k], err_msg=(mode, k))


@pytest.mark.parametrize("n,radius,kind,outside", [(8000, 0.25, nau.PERIODIC, 0),
                                                   (8000, 0.25, nau.SYMMETRIC, 0),
                                                   (24000, 0.25, nau.PERIODIC, 0),
                                                   (3000, 0.45, nau.SYMMETRIC, 0),
                                                   (3000, 0.25, nau.SYMMETRIC, 7)])
def test_neighbor_lists_capacity_growth_and_fallback(n, radius, kind, outside):
    """~1600 entries per list (capacity grows from 64 in one retry) and ~4700 (above
    the list cap: the step falls back to sweeping) give the sweep's results; so do
    the fp32 list pre-filter (radius 1.8 cells) and particles outside their cell
    box (fp16 pre-filter disabled at run time)."""
    build = _random_deck(n, 77, kind, radius, outside)
    for fast in (False, True):
        off, _ = _run_deck(build, fast, 0, 2)
        for mode in ((1, 2) if fast else (1,)):
            on, _ = _run_deck(build, fast, mode, 2)
            for k in on:
                np.testing.assert_array_equal(on[k], off[k], err_msg=(fast, mode, k))


# ------------------------------------------- device SFL evaluator (§8(f) 1) ----
def _vm_context():
    import sfl_mini
    z = np.load(os.path.join(GOLD, "vm_cases.npz"))
    meta = json.loads(str(z["meta"]))
    c = nau.Context(0)
    c.set_domain(3, [0, 0, 0], [2, 2, 2], [0.5, 0.5, 0.5], [nau.CUTOFF] * 3)
    c.set_particles(z["pos"])
    for k, (r, cc) in meta["shapes"].items():
        c.add_field(k, r, cc, z["f_" + k])
    for k, r in (("o1", 1), ("o2", 2), ("o3", 3)):
        c.add_field(k, r, 1, 0.0)
    c.add_field("o9", 3, 3, 0.0)
    sym = {k: ("field", c.fields[k].id) for k in meta["shapes"]}
    sym.update({k: ("const", np.array(v)) for k, v in meta["consts"].items()})
    return z, meta, c, sym, sfl_mini


def test_vm_expressions_vs_reference():
    """50 particle-wise SFL expressions (every operator, builtin and shape rule) through
    nau_eval vs the reference's own parser + AST evaluation: bitwise without a libm
    transcendental, within 1e-14 with one (CUDA vs glibc exp/log/sin/cos/tan/pow)."""
    z, meta, c, sym, sfl_mini = _vm_context()
    try:
        for idx, expr in enumerate(meta["expressions"]):
            want = z[f"e{idx}"]
            out = {1: "o1", 2: "o2", 3: "o3", 9: "o9"}[want.shape[0]]
            prog, res = sfl_mini.lower(expr, sym)
            c.eval_program(prog, res, out)
            got = c.download(out)
            if sfl_mini.uses_transcendental(expr):
                np.testing.assert_allclose(got, want, rtol=1e-14, atol=1e-300, err_msg=expr)
            else:
                np.testing.assert_array_equal(got, want, err_msg=expr)
        # rand: the reference's RandomState, fresh counters per expression; the last
        # expression drawn twice (counters persist across evaluations)
        for idx, expr in enumerate(meta["rand"]):
            c.set_random_state(meta["rand_seed"])
            want = z[f"r{idx}"]
            out = {1: "o1", 2: "o2"}[want.shape[0]]
            prog, res = sfl_mini.lower(expr, sym)
            c.eval_program(prog, res, out)
            np.testing.assert_array_equal(c.download(out), want, err_msg=expr)
            if f"r{idx}_again" in z:
                c.eval_program(prog, res, out)
                np.testing.assert_array_equal(c.download(out), z[f"r{idx}_again"], err_msg=expr)
                assert (c.random_counters() == 2).all()
    finally:
        c.close()


def test_vm_shape_errors_and_nan_audit():
    z, meta, c, sym, sfl_mini = _vm_context()
    try:
        msgs = json.loads(str(z["error_messages"]))
        for expr, ref_msg in zip(meta["errors"], msgs):
            prog, res = sfl_mini.lower(expr, sym)
            with pytest.raises(nau.NauError) as ei:
                c.eval_program(prog, res, "o9")
            assert ei.value.status == 1, expr  # NAU_ERR_RUNTIME
            assert ref_msg.startswith(ei.value.message), (expr, ei.value.message, ref_msg)
        # wrong LHS shape (case.cpp:41-44)
        prog, res = sfl_mini.lower("u", sym)
        with pytest.raises(nau.NauError, match="LHS field is 1x1 but RHS produced 3x1"):
            c.eval_program(prog, res, "o1")
        # NaN audit (case.cpp:46-53): log of a negative value, lowest original index
        prog, res = sfl_mini.lower("log(t)", sym)
        t = z["f_t"][0]
        with pytest.raises(nau.NauError) as ei:
            c.eval_program(prog, res, "o1")
            c.sync()
        assert ei.value.status == 2 and ei.value.particle == int(np.flatnonzero(t <= 0)[0])
    finally:
        c.close()


def test_vm_two_phase_and_inactive():
    """out may alias an operand (two-phase write); particles outside a cut-off
    domain are inactive and keep their value (case.cpp:36-40)."""
    z, meta, c, sym, sfl_mini = _vm_context()
    try:
        s0 = c.download("s").copy()
        t0 = c.download("t").copy()
        prog, res = sfl_mini.lower("s*s+t", sym)
        c.eval_program(prog, res, "s")
        np.testing.assert_array_equal(c.download("s"), s0 * s0 + t0)
    finally:
        c.close()
    c = nau.Context(0)
    try:
        pos = z["pos"].copy()
        pos[0, 7] = 1.5  # outside the [0, 1] cut-off box: deactivated by the shift
        c.set_domain(3, [0, 0, 0], [2, 2, 2], [0.5, 0.5, 0.5], [nau.CUTOFF] * 3)
        c.set_particles(pos)
        c.add_field("s", 1, 1, z["f_s"])
        c.add_field("o1", 1, 1, -7.0)
        c.boundary_shift()
        import sfl_mini
        prog, res = sfl_mini.lower("2*s", {"s": ("field", c.fields["s"].id)})
        c.eval_program(prog, res, "o1")
        got = c.download("o1")[0]
        want = 2 * z["f_s"][0]
        want[7] = -7.0
        np.testing.assert_array_equal(got, want)
    finally:
        c.close()


def test_async_host_io_matches_sync():
    """nau_upload_async / nau_download_async (double-buffered staging on copy
    streams) give the same per-step results as the synchronous calls."""
    import torch
    sc = scenes.dam_break(2)
    outs = {}
    for mode in ("sync", "async"):
        c = nau.Context(0)
        try:
            p = _gpu_dam(c, sc)
            h_r = torch.from_numpy(np.ascontiguousarray(sc.pos)).pin_memory()
            h_v = torch.from_numpy(0.01 * np.ones((2, sc.n))).pin_memory()
            res = []
            for s in range(4):
                bufs = {k: torch.empty((r, sc.n), dtype=torch.float64).pin_memory()
                        for k, r in (("r", 2), ("v", 2), ("rho", 1))}
                if mode == "sync":
                    c.upload_ptr("r", h_r.data_ptr())
                    c.upload_ptr("v", h_v.data_ptr())
                    c.wcsph_step(p)
                    for k, t in bufs.items():
                        c.download_ptr(k, t.data_ptr())
                else:
                    c.upload_async("r", h_r.data_ptr())
                    c.upload_async("v", h_v.data_ptr())
                    c.wcsph_step(p)
                    for k, t in bufs.items():
                        c.download_async(k, t.data_ptr())
                res.append(bufs)
            c.sync()
            outs[mode] = [{k: t.numpy().copy() for k, t in b.items()} for b in res]
        finally:
            c.close()
    for a, b in zip(outs["sync"], outs["async"]):
        for k in a:
            np.testing.assert_array_equal(a[k], b[k], err_msg=k)


# ------------------------------------------------------- slab primitives ----
def test_select_pack_load_roundtrip(ctx):
    import torch
    rng = np.random.default_rng(21)
    spec = cases.random_spec(rng, dim=3, n=5000, kinds=[0, 1, 2], cells=[5, 4, 3])
    spec["fields"]["gid"] = (np.arange(5000)[::-1].astype(np.float64) * 3).reshape(1, -1)
    cases.gpu_context(spec, ctx)
    W = ctx.L.nau_row_width(ctx.h)
    assert W == 3 + 1 + 3 + 1 + 1 + 1 + 1
    slots = torch.empty(5000, dtype=torch.int32, device="cuda")
    import ctypes as C
    cnt = C.c_long(0)
    assert ctx.L.nau_select(ctx.h, 0, 1.0, 3.0, -1, 0.0, 0.0, slots.data_ptr(), C.byref(cnt)) == 0
    cx = np.floor(spec["pos"][0] / 0.3).astype(int) % 5
    assert cnt.value == int(((cx >= 1) & (cx < 3)).sum())
    rows = torch.empty((cnt.value, W), dtype=torch.float64, device="cuda")
    assert ctx.L.nau_pack_rows(ctx.h, slots.data_ptr(), cnt.value, rows.data_ptr()) == 0
    h = rows.cpu().numpy()
    sel = np.nonzero((cx >= 1) & (cx < 3))[0]
    # columns: r(3) A V(3) rho M Rp gid -> gid is the last column here
    exp = np.concatenate([spec["pos"], spec["fields"]["A"], spec["fields"]["V"],
                          spec["fields"]["rho"], spec["fields"]["M"], spec["fields"]["Rp"],
                          spec["fields"]["gid"]], axis=0).T[sel]
    np.testing.assert_array_equal(h[np.argsort(h[:, -1])], exp[np.argsort(exp[:, -1])])
    # reload only those rows keyed by gid: cells list them in ascending gid
    assert ctx.L.nau_load_rows(ctx.h, rows.data_ptr(), cnt.value, ctx.fields["gid"].id) == 0
    ctx.n = cnt.value
    _, start, count, srt = ctx.cell_tables()
    gid_of_local = ctx.download("gid")[0]
    for c in np.nonzero(count)[0][:50]:
        g = gid_of_local[srt[start[c]:start[c] + count[c]]]
        assert np.all(np.diff(g) > 0)


def test_slab_path_single_rank_matches_plain(ctx):
    """The slab driver (select/pack/load every step) on one GPU = the plain path, bitwise."""
    import bench
    from paper_1710_08259_b200 import slab as slab_mod

    class D:
        world, rank, local, pg = 1, 0, 0, None

    plain = bench.DamBreak(2)
    plain.sc = scenes.dam_break(2, dx=0.05, fluid=(1.0, 1.0), tank=(2.0, 1.6))
    plain.sc.fields["v"][0, : plain.sc.params["n_fluid"]] = 3.0
    ctx.set_mode(False)
    plain.setup(ctx)
    for _ in range(8):
        plain.step(ctx)
    ref_r, ref_v = ctx.download("r"), ctx.download("v")
    ctx2 = nau.Context(0)
    sl = bench.DamBreakSlab(2, D())
    sl.sc = plain.sc = scenes.dam_break(2, dx=0.05, fluid=(1.0, 1.0), tank=(2.0, 1.6))
    sl.sc.fields["v"][0, : sl.sc.params["n_fluid"]] = 3.0
    sl.setup(ctx2)
    for _ in range(8):
        sl.step(ctx2)
    gid = ctx2.download("gid")[0].astype(int)
    r2, v2 = np.empty_like(ref_r), np.empty_like(ref_v)
    r2[:, gid], v2[:, gid] = ctx2.download("r"), ctx2.download("v")
    np.testing.assert_array_equal(r2, ref_r)
    np.testing.assert_array_equal(v2, ref_v)
    ctx2.close()


class _Hub:
    """In-process rendezvous for slab ranks run as host threads on one GPU: each rank has
    its own context and stream; rows meet on the host side (no kernel waits on another
    rank's kernel), so the multi-rank SlabRank logic runs on the real CUDA backend."""

    def __init__(self, world):
        import threading
        self.world, self.bar, self.box = world, threading.Barrier(world, timeout=120), {}


class _ThreadExchanger:
    """slab.Exchanger's contract (swap / allreduce_sum) over a _Hub."""

    def __init__(self, hub, rank, periodic, device):
        w = hub.world
        self.hub, self.rank, self.world, self.periodic, self.device = hub, rank, w, periodic, device
        self.left = (rank - 1) % w if (periodic or rank > 0) else None
        self.right = (rank + 1) % w if (periodic or rank < w - 1) else None

    def swap(self, to_left, to_right, width):
        import torch
        h = self.hub
        torch.cuda.synchronize()  # blocks come from other contexts' streams
        h.box[(self.rank, "L")] = to_left
        h.box[(self.rank, "R")] = to_right
        h.bar.wait()
        empty = torch.empty((0, width), dtype=torch.float64, device=self.device)

        def take(src, side):
            if src is None:
                return None
            t = h.box.get((src, side))
            return empty if t is None else t.clone()
        fl, fr = take(self.left, "R"), take(self.right, "L")
        torch.cuda.synchronize()
        h.bar.wait()
        return fl, fr

    def allreduce_sum(self, t):
        h = self.hub
        h.box[(self.rank, "sum")] = t.clone()
        h.bar.wait()
        tot = sum(h.box[(r, "sum")].cpu() for r in range(self.world))
        h.bar.wait()
        t.copy_(tot.to(t.device))
        return t


@pytest.mark.parametrize("fast", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_slab_ranks_with_rebalancing_match_plain(ctx, world, fast):
    """SURVEY.md §8(e) on the CUDA backend: `world` slab ranks (threads, one context each,
    one GPU) from skewed bounds with migration, ghost refresh and re-balancing every 3
    steps; owned particles gathered by global id = the single-context path, bitwise."""
    import threading

    import bench
    from paper_1710_08259_b200 import slab as slab_mod

    def scene():
        sc = scenes.dam_break(2, dx=0.05, fluid=(1.0, 1.0), tank=(2.0, 1.6))
        sc.fields["v"][0, : sc.params["n_fluid"]] = 6.0
        return sc

    steps = 9
    plain = bench.DamBreak(2)
    plain.sc = scene()
    ctx.set_mode(fast)  # FAST: the paired-list kernels with ghosts in the lists
    plain.setup(ctx)
    for _ in range(steps):
        plain.step(ctx)
    ref_r, ref_v = ctx.download("r"), ctx.download("v")
    ctx.set_mode(False)
    hub = _Hub(world)
    out, errs, drv = {}, [], {}

    def rank_main(rank):
        try:
            class D:
                pg = None
            D.world, D.rank, D.local = world, rank, 0
            c = nau.Context(0)
            c.set_mode(fast)
            sl = bench.DamBreakSlab(2, D())
            sl.sc = scene()
            sl.setup(c)
            sc = sl.sc
            R = sc.params["radius"]
            lo, hi = sc.min_cells[0] * sc.cell_size[0], sc.max_cells[0] * sc.cell_size[0]
            # skewed start (2R-wide slabs, one huge): re-balancing must move bounds past
            # whole slabs, so particles hop over a rank
            skew = [lo + 2 * R * i for i in range(world)] + [hi]
            import torch
            rows = slab_mod.initial_rows(sc, sl.FIELDS, skew, rank, R, False)
            sl.backend.load(torch.from_numpy(rows).to(sl.backend.device))
            ex = _ThreadExchanger(hub, rank, False, sl.backend.device)
            r = slab_mod.SlabRank(sl.backend, ex, skew, R, False, rebalance_every=3, nbins=256)
            drv[rank] = r
            for _ in range(steps):
                r.step()
            own = c.download("ghost")[0] == 0
            out[rank] = (c.download("gid")[0][own].astype(int), c.download("r")[:, own],
                         c.download("v")[:, own])
            c.close()
        except BaseException as e:  # surface thread failures in the test
            errs.append(e)
            hub.bar.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    assert all(drv[r].rebalances >= 1 for r in range(world)), "bounds never changed"
    gid = np.concatenate([out[r][0] for r in range(world)])
    assert np.array_equal(np.sort(gid), np.arange(ref_r.shape[1])), "a particle lost or owned twice"
    r2, v2 = np.empty_like(ref_r), np.empty_like(ref_v)
    for r in range(world):
        r2[:, out[r][0]], v2[:, out[r][0]] = out[r][1], out[r][2]
    np.testing.assert_array_equal(r2, ref_r)
    np.testing.assert_array_equal(v2, ref_v)


def test_native_slab_exchange_single_rank_matches_plain(ctx):
    """nau_comm_init / nau_migrate / nau_halo_exchange (comm.cu, NCCL bound at run
    time) on one rank: the step loop through the native exchange = the plain path,
    bitwise (same check as the torch.distributed driver above)."""
    import bench

    class D:
        world, rank, local, pg = 1, 0, 0, None

    sc_args = dict(dx=0.05, fluid=(1.0, 1.0), tank=(2.0, 1.6))
    plain = bench.DamBreak(2)
    plain.sc = scenes.dam_break(2, **sc_args)
    plain.sc.fields["v"][0, : plain.sc.params["n_fluid"]] = 3.0
    ctx.set_mode(False)
    plain.setup(ctx)
    for _ in range(8):
        plain.step(ctx)
    ref_r, ref_v = ctx.download("r"), ctx.download("v")
    ctx2 = nau.Context(0)
    sl = bench.DamBreakSlab(2, D(), native=True)
    sl.sc = scenes.dam_break(2, **sc_args)
    sl.sc.fields["v"][0, : sl.sc.params["n_fluid"]] = 3.0
    sl.setup(ctx2)
    for _ in range(8):
        sl.step(ctx2)
    gid = ctx2.download("gid")[0].astype(int)
    r2, v2 = np.empty_like(ref_r), np.empty_like(ref_v)
    r2[:, gid], v2[:, gid] = ctx2.download("r"), ctx2.download("v")
    np.testing.assert_array_equal(r2, ref_r)
    np.testing.assert_array_equal(v2, ref_v)
    ctx2.close()


def test_native_comm_swap_on_a_one_rank_ring():
    """nau_comm_swap through real NCCL send/recv: on a 1-rank periodic ring both
    neighbours are this rank, so (posting order, slab.py Exchanger.swap) the block
    sent left comes back from the right and vice versa; empty blocks too."""
    import torch
    c = nau.Context(0)
    try:
        c.set_domain(1, [0], [4], [0.25], [nau.PERIODIC])
        c.set_particles(np.array([[0.1, 0.4, 0.6, 0.9]]))
        c.add_field("gid", 1, 1, np.arange(4.0))
        c.add_field("ghost", 1, 1, 0.0)
        c.comm_init(nau.Context.comm_unique_id(), 1, 0)
        c.slab_config(0, [0.0, 1.0], True, 0.25)
        assert c.slab_bounds() == [0.0, 1.0]
        a = torch.arange(21, dtype=torch.float64, device="cuda").reshape(7, 3)
        b = -torch.arange(6, dtype=torch.float64, device="cuda").reshape(2, 3)
        fl, fr = c.comm_swap(a, b)
        assert torch.equal(fr, a) and torch.equal(fl, b)
        fl, fr = c.comm_swap(b[:0], a)
        assert fr.shape == (0, 3) and torch.equal(fl, a)
        with pytest.raises(nau.NauError):  # bounds must rise
            c.slab_config(0, [1.0, 0.0], True, 0.25)
    finally:
        c.close()


# ------------------------------------------------------------- DEM / n-body ----
def _dem_port_step(ps, st, prm, R, m):
    """vdot = dem_lsd(v,R,kn,en,m,cf,Rs) + g; v = euler(v,vdot,dt); r = euler(r,v,dt); shift."""
    act = ps.active.astype(bool)
    if ps.tables is None:
        ps.build_cells()
    acc = ps.interact(port.DEM_LSD, [st["v"], R, prm["kn"], prm["en"], m, prm["cf"],
                                     prm["search_radius"]], (3, 1))
    g = np.asarray(prm["g"]).reshape(3, 1)
    st["vdot"][:, act] = acc[:, act] + g
    st["v"][:, act] = st["v"][:, act] + prm["dt"] * st["vdot"][:, act]
    ps.pos[:, act] = ps.pos[:, act] + prm["dt"] * st["v"][:, act]
    ps.boundary_shift()
    ps.tables = None


@pytest.mark.parametrize("fast", [False, True])
def test_dem_deck_vs_port(ctx, fast):
    """cfg3 deck on a small compressed column (many contacts, floor via mirror images):
    EXACT mode bitwise (no libm transcendental in the linear law); FAST within 1e-10."""
    sc = scenes.dem_column(n=6000, box=(0.03, 0.03, 0.06), dt=1e-5, placement="lattice")
    prm = sc.params
    sc.pos[2] *= 0.6  # squeeze the column vertically: overlapping contacts from step 1
    sc.fields["v"][:] = np.random.default_rng(3).uniform(-0.05, 0.05, (3, sc.n))
    ctx.set_mode(fast)
    ctx.set_domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
    ctx.set_particles(sc.pos)
    for k in ("v", "vdot", "R", "m"):
        ctx.add_field(k, np.asarray(sc.fields[k]).reshape(-1, sc.n).shape[0], 1, sc.fields[k])
    ctx.boundary_shift()
    p = nau.DemParams()
    f = ctx.fields
    p.law, p.f_v, p.f_vdot, p.f_R, p.f_m = 8, f["v"].id, f["vdot"].id, f["R"].id, f["m"].id
    p.P, p.Q, p.cf, p.search_radius, p.dt = prm["kn"], prm["en"], prm["cf"], prm["search_radius"], prm["dt"]
    for a in range(3):
        p.g[a] = prm["g"][a]
    dom = port.Domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
    ps = port.ParticleSystem(dom, sc.pos)
    ps.boundary_shift()
    st = {"v": sc.fields["v"].copy(), "vdot": np.zeros((3, sc.n))}
    for s in range(5):
        ctx.dem_step(p)
        _dem_port_step(ps, st, prm, sc.fields["R"], sc.fields["m"])
    assert np.abs(st["vdot"][2] - prm["g"][2]).max() > 1.0, "no contact forces: test is vacuous"
    for k, ref_v in (("r", ps.pos), ("v", st["v"]), ("vdot", st["vdot"])):
        got = ctx.download(k)
        if fast:
            assert rel_err(got, ref_v) <= TOL_STEP, k
        else:
            np.testing.assert_array_equal(got, ref_v, err_msg=k)
    ctx.set_mode(False)


@pytest.mark.parametrize("fast", [False, True])
def test_gravity_leapfrog_vs_port(ctx, fast):
    """cfg4 deck on N = 1024 Plummer bodies: 3 leapfrog steps within 1e-10 (pow vs r^1.5);
    total momentum stays ~0. FAST runs the multi-body kernel (uniform G, eps > 0)."""
    sc = scenes.plummer(n=1024)
    prm = sc.params
    ctx.set_mode(fast)
    ctx.set_domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
    ctx.set_particles(sc.pos)
    ctx.add_field("v", 3, 1, sc.fields["v"])
    ctx.add_field("a", 3, 1, 0.0)
    ctx.boundary_shift()
    ctx.interact("nbody_gravity", [prm["m"], prm["G"], prm["eps"]], "a")
    p = nau.GravityParams()
    p.f_v, p.f_a, p.f_m = ctx.fields["v"].id, ctx.fields["a"].id, -1
    p.m, p.G, p.eps, p.dt = prm["m"], prm["G"], prm["eps"], prm["dt"]
    dom = port.Domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
    ps = port.ParticleSystem(dom, sc.pos)
    ps.boundary_shift()
    v = sc.fields["v"].copy()
    grav = lambda: ps.interact(port.GRAVITY, [prm["m"], prm["G"], prm["eps"]], (3, 1))
    a = grav()
    for s in range(3):
        ctx.leapfrog_step(p)
        v = v + (0.5 * prm["dt"]) * a
        ps.pos = ps.pos + prm["dt"] * v
        ps.tables = None
        a = grav()
        v = v + (0.5 * prm["dt"]) * a
    assert rel_err(ctx.download("r"), ps.pos) <= TOL_STEP
    assert rel_err(ctx.download("v"), v) <= TOL_STEP
    assert rel_err(ctx.download("a"), a) <= TOL_STEP
    mom = ctx.download("v").sum(axis=1) * prm["m"]
    assert np.abs(mom).max() <= 1e-12
    ctx.set_mode(False)


@pytest.mark.parametrize("fast", [False, True])
def test_gravity_shard_path_matches_plain(ctx, fast):
    """The sharded n-body path (pack sources -> [all-gather] -> gravity vs sources) on one
    rank = the plain leapfrog, bitwise (same global source order)."""
    import bench

    class D:
        world, rank, local, pg = 1, 0, 0, None

    plain = bench.Gravity.__new__(bench.Gravity)
    plain.sc = scenes.plummer(n=2048)
    ctx.set_mode(fast)
    plain.setup(ctx)
    for _ in range(3):
        plain.step(ctx)
    ref = {k: ctx.download(k) for k in ("r", "v", "a")}
    ctx2 = nau.Context(0)
    ctx2.set_mode(fast)
    sh = bench.GravityShard.__new__(bench.GravityShard)
    sh.dist = D()
    sh.sc = scenes.plummer(n=2048)
    sh.setup(ctx2)
    for _ in range(3):
        sh.step(ctx2)
    for k in ("r", "v", "a"):
        np.testing.assert_array_equal(ctx2.download(k), ref[k], err_msg=k)
    ctx.set_mode(False)
    ctx2.close()


@pytest.mark.parametrize("fast", [False, True])
def test_gravity_source_chunks_continue_the_sums(ctx, fast):
    """nau_gravity_sources_part over 4 source chunks in global order (what the broadcast
    pipeline of the sharded step consumes) = one nau_gravity_sources call, bitwise."""
    import torch
    sc = scenes.plummer(n=2048)
    prm = sc.params
    ctx.set_mode(fast)
    ctx.set_domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
    ctx.set_particles(sc.pos)
    ctx.add_field("a", 3, 1, 0.0)
    ctx.add_field("b", 3, 1, 0.0)
    ctx.boundary_shift()
    rows = torch.empty((sc.n, 4), dtype=torch.float64, device="cuda:0")
    ctx._check(ctx.L.nau_pack_sources(ctx.h, -1, prm["m"], rows.data_ptr()))
    fa, fb = ctx.fields["a"].id, ctx.fields["b"].id
    ctx._check(ctx.L.nau_gravity_sources(ctx.h, rows.data_ptr(), sc.n, 0, prm["G"], prm["eps"], fa))
    nc = sc.n // 4
    for c in range(4):
        chunk = rows[c * nc:(c + 1) * nc]
        ctx._check(ctx.L.nau_gravity_sources_part(ctx.h, chunk.data_ptr(), nc, -c * nc, prm["G"],
                                                  prm["eps"], fb, int(c > 0)))
    ctx.sync()
    np.testing.assert_array_equal(ctx.download("b"), ctx.download("a"))
    ctx.set_mode(False)


def test_list_stats_of_the_paired_lists():
    """nau_list_stats on the FAST dam-break deck: one walker per particle pair, the union
    lists hold every neighbour of both particles (entries >= the larger neighbour count,
    <= their sum) and the warp-wide walk loses little to uneven lists."""
    c = nau.Context(0)
    try:
        sc = scenes.dam_break(3, dx=0.04)
        p = _gpu_dam(c, sc)
        c.set_mode(True)
        c.wcsph_step(p)
        c.sync()
        assert c.wcsph_path["source"] == "paired"
        c.wcsph_pass(p, 0)  # the lists of the current positions
        st = c.list_stats()
        counts = c.neighbor_counts(sc.params["radius"])
        n_act = int(c.active().sum())
        assert st["walkers"] == (n_act + 1) // 2
        assert counts.sum() / 2.0 <= st["entries"] <= counts.sum() * 1.02
        assert 0.8 < st["lane_efficiency"] <= 1.0
    finally:
        c.close()


# ------------------------------------------------ graphs / async lists ----
@pytest.mark.parametrize("fast", [False, True])
@pytest.mark.parametrize("deck", ["dam3d", "random_overflow"])
def test_graph_replay_equals_plain_steps(fast, deck):
    """nau_wcsph_step without host synchronisation and replayed as CUDA graphs after two
    warm-up calls equals the plain step loop bitwise over 9 steps — including a deck
    whose neighbour lists overflow (capacity 64 -> grown from the published overflow,
    overflowed slots swept by the fallback pass) and one above the list cap (every
    step falls back for the long lists)."""
    if deck == "dam3d":
        build = lambda c: _gpu_dam(c, scenes.dam_break(3, dx=0.04))
    else:
        build = _random_deck(24000, 2, nau.PERIODIC, 0.25)
    runs = []
    for graphs in (False, True):
        c = nau.Context(0)
        try:
            p = build(c)
            c.set_mode(fast)
            c.set_graphs(graphs)
            for _ in range(9):
                c.wcsph_step(p)
            c.sync()
            runs.append(({k: c.download(k) for k in ("r", "rho", "p", "v", "vdot")}, c.active()))
        finally:
            c.close()
    np.testing.assert_array_equal(runs[0][1], runs[1][1])
    for k in runs[0][0]:
        np.testing.assert_array_equal(runs[1][0][k], runs[0][0][k], err_msg=k)
