"""CPU pins of the device SFL evaluator's program semantics.

tests/golden/vm_cases.npz holds the reference's own evaluation (sfl parser +
AST + Tensor operators, oracle/_ref via nref_eval) of 50 expressions over random
fields of every shape class. The lowering in sfl_mini.py and its host
interpreter must reproduce them: bitwise without a libm transcendental, to
1e-14 relative with one (numpy's exp/log/sin/pow vs glibc).
"""
import json
import os

import numpy as np
import pytest

import sfl_mini

GOLD = os.path.join(os.path.dirname(__file__), "golden", "vm_cases.npz")


def _load():
    z = np.load(GOLD)
    meta = json.loads(str(z["meta"]))
    names = list(meta["shapes"])
    fields = {j: (meta["shapes"][k][0], meta["shapes"][k][1], z["f_" + k]) for j, k in enumerate(names)}
    sym = {k: ("field", j) for j, k in enumerate(names)}
    sym.update({k: ("const", np.array(v)) for k, v in meta["consts"].items()})
    return z, meta, fields, sym


def test_vm_golden_has_all_shape_classes():
    z, meta, fields, sym = _load()
    shapes = {tuple(v) for v in meta["shapes"].values()}
    assert shapes == {(1, 1), (3, 1), (3, 3)}
    assert len(meta["expressions"]) >= 50


@pytest.mark.parametrize("idx", range(50))
def test_lowering_matches_reference(idx):
    z, meta, fields, sym = _load()
    expr = meta["expressions"][idx]
    prog, res = sfl_mini.lower(expr, sym)
    n = z["pos"].shape[1]
    got = sfl_mini.run_numpy(prog, res, fields, n)
    want = z[f"e{idx}"]
    assert got.shape == want.shape, expr
    if sfl_mini.uses_transcendental(expr):
        np.testing.assert_allclose(got, want, rtol=1e-14, atol=0, err_msg=expr)
    else:
        np.testing.assert_array_equal(got, want, err_msg=expr)


def test_error_cases_are_reference_errors():
    z, meta, fields, sym = _load()
    msgs = json.loads(str(z["error_messages"]))
    assert all(m for m in msgs), msgs  # every listed program is rejected by the reference


def test_rand_matches_reference_random_state():
    """rand(a, b) = RandomState::uniform(i, a, b) with per-particle draw counters
    (sfl/random_state.hpp); counters persist across evaluations."""
    z, meta, fields, sym = _load()
    n = z["pos"].shape[1]
    seed = meta["rand_seed"]
    for idx, expr in enumerate(meta["rand"]):
        prog, res = sfl_mini.lower(expr, sym)
        counters = np.zeros(n, dtype=np.uint64)
        got = sfl_mini.run_numpy(prog, res, fields, n, seed=seed, counters=counters)
        np.testing.assert_array_equal(got, z[f"r{idx}"], err_msg=expr)
        if f"r{idx}_again" in z:
            got2 = sfl_mini.run_numpy(prog, res, fields, n, seed=seed, counters=counters)
            np.testing.assert_array_equal(got2, z[f"r{idx}_again"], err_msg=expr)
            assert not np.array_equal(got2, got)
