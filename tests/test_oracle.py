"""CPU tests: the oracle itself, pinned against the reference.

* oracle/port (C restatement) == golden fixtures made by the reference, bitwise;
* oracle/port == oracle/_ref live on fresh random cases (when the reference build exists);
* the reference's own unit tests pass on the shim build (pins the Eigen shim);
* kernel known-answer tests from /root/reference/proj/tests/test_kernel.cpp:46-108;
* the input generator's RNG == the reference RandomState.
"""
import json
import math
import os
import subprocess

import numpy as np
import pytest

import cases
import deck_oracle
from oracle import port, ref
from paper_1710_08259_b200 import scenes

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


def unpack_spec(z, p):
    meta = json.loads(str(z[p + "meta"]))
    spec = {k: meta[k] for k in ("dim", "min_cells", "max_cells", "cell_size", "kinds")}
    spec["consts"] = meta["consts"]
    spec["pos"] = z[p + "pos"]
    spec["fields"] = {k: z[p + "f_" + k] for k in meta["fields"]}
    return spec


def golden_cases():
    z = load("random_cases.npz")
    return z, int(z["n_random_cases"])


@pytest.mark.parametrize("idx", range(16))
def test_port_matches_golden(idx):
    z, n = golden_cases()
    if idx >= n:
        pytest.skip("no such case")
    p = f"c{idx}_"
    spec = unpack_spec(z, p)
    ps = cases.port_system(spec)
    cell_of, start, cnt, srt = ps.tables
    np.testing.assert_array_equal(cell_of, z[p + "cell_of"])
    np.testing.assert_array_equal(start, z[p + "cell_start"])
    np.testing.assert_array_equal(cnt, z[p + "cell_count"])
    np.testing.assert_array_equal(srt, z[p + "sorted"])
    np.testing.assert_array_equal(ps.neighbor_counts(spec["consts"]["R"]), z[p + "counts"])
    for k, entry in enumerate(cases.op_list(spec["dim"])):
        if p + f"op{k}_error" in z:
            with pytest.raises(port.OracleError):
                cases.port_eval(spec, ps, entry)
            continue
        got = cases.port_eval(spec, ps, entry)
        # bitwise: same operation order as the reference, no FMA, same libm
        np.testing.assert_array_equal(got, z[p + f"op{k}"], err_msg=f"{entry[0]} {entry[2]}")


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built here")
@pytest.mark.parametrize("seed", range(6))
def test_port_matches_reference_live(seed):
    rng = np.random.default_rng(1000 + seed)
    spec = cases.random_spec(rng, n=int(rng.integers(50, 300)))
    ps = cases.port_system(spec)
    rc = cases.ref_case(spec)
    nc = int(np.prod(spec["max_cells"]))
    for a, b in zip(ps.tables, rc.cell_tables(nc)):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(ps.neighbor_counts(0.3), rc.neighbor_counts(0.3))
    for entry in cases.op_list(spec["dim"]):
        np.testing.assert_array_equal(cases.port_eval(spec, ps, entry),
                                      cases.ref_eval(spec, rc, entry), err_msg=entry[0])


@pytest.mark.skipif(not os.path.exists(ref.UNIT_PATH), reason="oracle/_ref not built here")
def test_reference_unit_tests_pass_on_shim_build():
    r = subprocess.run([ref.UNIT_PATH], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failed" in r.stdout


def test_dam_break_deck_port_matches_reference_golden():
    z = load("dam_break_2d_small.npz")
    meta = json.loads(str(z["dam_meta"]))
    sc = scenes.dam_break(2, dx=meta["dx"], fluid=tuple(meta["fluid"]), tank=tuple(meta["tank"]))
    ps, st = deck_oracle.make_system(sc)
    for s in range(1, meta["steps"] + 1):
        deck_oracle.step(ps, st, sc.params)
        if s in (1, meta["steps"]):
            np.testing.assert_array_equal(ps.pos, z[f"dam_s{s}_r"])
            for k in ("rho", "p", "v", "vdot"):
                np.testing.assert_array_equal(st[k], z[f"dam_s{s}_{k}"], err_msg=k)
            np.testing.assert_array_equal(ps.active, z[f"dam_s{s}_active"])


def test_microbench_port_matches_golden():
    z = load("microbench_small.npz")
    sc = scenes.sph_microbench(n=int(z["mb_n"]))
    prm = sc.params
    dom = port.Domain(3, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
    ps = port.ParticleSystem(dom, sc.pos)
    ps.boundary_shift()
    ps.build_cells()
    np.testing.assert_array_equal(ps.tables[1], z["mb_cell_start"])
    np.testing.assert_array_equal(ps.tables[3], z["mb_sorted"])
    np.testing.assert_array_equal(ps.neighbor_counts(prm["radius"]), z["mb_counts"])
    A = sc.fields["A"]
    for fam, sfx in ((port.K_WENDLAND, "w"), (port.K_CUBIC, "c")):
        rho = ps.interact(port.SPH_S, [1.0, prm["mass"], 1.0, prm["radius"]], (1, 1), kfamily=fam)
        np.testing.assert_array_equal(rho, z["mb_rho_" + sfx])
        rho_w = z["mb_rho_w"]  # the reference uses the Wendland density for G and L
        G = ps.interact(port.SPH_G11, [A, prm["mass"], rho_w, prm["radius"]], (3, 1), kfamily=fam)
        L = ps.interact(port.SPH_L0, [A, prm["mass"], rho_w, prm["radius"]], (1, 1), kfamily=fam)
        np.testing.assert_array_equal(G, z["mb_G_" + sfx])
        np.testing.assert_array_equal(L, z["mb_L_" + sfx])


def test_rng_matches_reference_random_state():
    z = load("rng.npz")
    d = z["draws"]
    np.testing.assert_array_equal(port.uniform_draws(int(z["seed"]), d.shape[1], d.shape[0]), d)
    np.testing.assert_array_equal(scenes.uniform_draws(int(z["seed"]), d.shape[1], d.shape[0]), d)


# ---- kernel KATs: /root/reference/proj/tests/test_kernel.cpp ----
def quadrature(fam, kdim, h):
    n = 10000
    a, b = 0.0, 2.0 * h
    def f(r):
        w = port.kernel_value(fam, kdim, h, r)
        return {1: 2.0 * w, 2: 2.0 * math.pi * r * w}.get(kdim, 4.0 * math.pi * r * r * w)
    hh = (b - a) / n
    s = f(a) + f(b)
    for i in range(1, n):
        s += f(a + i * hh) * (4.0 if i % 2 else 2.0)
    return s * hh / 3.0


def test_kernel_value_at_origin_and_support():  # test_kernel.cpp:46-53
    assert port.kernel_value(port.K_WENDLAND, 2, 0.25, 0.0) == pytest.approx(8.91268, rel=2e-5)
    assert port.kernel_value(port.K_WENDLAND, 2, 0.25, 0.5) == 0.0
    assert port.kernel_value(port.K_WENDLAND, 2, 0.25, 0.75) == 0.0
    # cubic spline (new): W(0) = sigma_d, sigma_3 = 1/(pi h^3)
    assert port.kernel_value(port.K_CUBIC, 3, 0.1, 0.0) == pytest.approx(1.0 / (math.pi * 1e-3))
    assert port.kernel_value(port.K_CUBIC, 3, 0.1, 0.2) == 0.0


@pytest.mark.parametrize("fam", [port.K_WENDLAND, port.K_CUBIC])
def test_kernel_normalisation(fam):  # test_kernel.cpp:55-62
    for kdim, h in ((1, 0.3), (2, 0.25), (3, 0.1)):
        assert quadrature(fam, kdim, h) == pytest.approx(1.0, abs=1e-3)


@pytest.mark.parametrize("fam", [port.K_WENDLAND, port.K_CUBIC])
def test_kernel_derivative_matches_finite_difference(fam):  # test_kernel.cpp:64-81
    h = 0.25
    rng = np.random.default_rng(21)
    for r in rng.uniform(1e-3, 2 * h - 1e-3, 20):
        eps = 1e-6 * h
        fd = (port.kernel_value(fam, 2, h, r + eps) - port.kernel_value(fam, 2, h, r - eps)) / (2 * eps)
        an = port.kernel_dq(fam, 2, h, r / h) / h
        assert abs(an - fd) <= 1e-6 * max(1.0, abs(an))


@pytest.mark.parametrize("fam", [port.K_WENDLAND, port.K_CUBIC])
def test_kernel_monotone(fam):  # test_kernel.cpp:98-108
    prev = port.kernel_value(fam, 3, 0.1, 0.0)
    for s in range(1, 401):
        w = port.kernel_value(fam, 3, 0.1, 2 * 0.1 * s / 400)
        assert w >= 0.0 and w <= prev + 1e-15
        prev = w


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built here")
def test_wendland_matches_reference_kernel():
    for kw, kdim in (("Wp51220", 1), ("Wp52220", 2), ("Wp53220", 3)):
        for d in np.linspace(0, 0.6, 37):
            assert port.kernel_value(port.K_WENDLAND, kdim, 0.25, d) == ref.kernel_value(kw, 0.25, d)


def test_lsd_restitution_head_on():
    """Linear spring-dashpot law (new; parity unpinned by the reference): two equal
    spheres colliding head-on rebound with the configured restitution 0.5
    (the analytic result of the damping ratio used), cf. test_interactions.cpp:332-357."""
    R, kn, en, m = 1e-3, 1e5, 0.5, 2500 * 4 / 3 * math.pi * 1e-9
    dom = port.Domain(3, [0, 0, 0], [8, 8, 8], [2.5e-3] * 3, [2, 2, 2])
    x = np.array([[0.009, 0.011], [0.01, 0.01], [0.01, 0.01]])  # just touching
    v = np.array([[0.5, -0.5], [0.0, 0.0], [0.0, 0.0]])
    dt = 1e-8 * 10
    for _ in range(6000):
        ps = port.ParticleSystem(dom, x)
        a = ps.interact(port.DEM_LSD, [v, R, kn, en, m, 0.0, 2 * R], (3, 1))
        v = v + dt * a
        x = x + dt * v
    assert v[0, 1] - v[0, 0] == pytest.approx(0.5 * 1.0, rel=2e-3)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_deck_fixtures_rebuild_through_the_public_api():
    """tests/golden/decks.npz (the reference's shipped decks, assembled by assemble_case)
    rebuilt through the reference's public API (Workspace fields, constants, variables,
    parsed equations — what tests/test_gpu_binding.py hands to GpuCase) steps bitwise
    like the assembled decks."""
    import json
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "decks.npz"))
    for deck in json.loads(str(Z["index"]))["decks"]:
        meta = json.loads(str(Z[f"{deck}_meta"]))
        d = meta["domain"]
        rc = ref.RefCase(d["dim"], d["min_cells"], d["max_cells"], d["cell_size"], d["kinds"],
                         Z[f"{deck}_s0_r"], seed=meta["seed"])
        for name, shape in meta["fields"]:
            if name != "r":
                rc.field(name, Z[f"{deck}_s0_{name}"], rows=shape[0], cols=shape[1])
        for name, v in meta["constants"]:
            rc.constant(name, np.array(v))
        for name, v in meta["variables"]:
            rc.variable(name, np.array(v))
        for name, text in meta["equations"]:
            rc.equation(name, text)
        for s in range(1, max(meta["steps"]) + 1):
            rc.solve_step(1)
            if s in meta["steps"]:
                for name, _ in meta["fields"]:
                    np.testing.assert_array_equal(rc.get(name), Z[f"{deck}_s{s}_{name}"],
                                                  err_msg=f"{deck} step {s} {name}")
