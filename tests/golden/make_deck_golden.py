"""Generate tests/golden/decks.npz: the reference's own shipped decks run by the
reference itself (oracle/_ref: the unmodified sources), as fixtures for the device
equation executor (nau_case_*, csrc/executor.cpp; tests/test_gpu_executor.py).

Run here, where /root/reference exists (the GPU box has only the fixtures):
    python tests/golden/make_deck_golden.py

Per deck (/root/reference/proj/tests/decks/<name>.yaml, parsed with PyYAML into the
CaseDocument bindings the reference's yaml-cpp reader would produce; assembled by
the reference's assemble_case with seed 7):
  meta       domain, constants and variables (values), fields (shapes), equations in
             the reference's canonical printed form (Equation::to_text), rand seed
  s0_*       every field after assembly (positions included), rand counters
  s<k>_*     every field, the active flags and every variable after k solve_step calls
Error cases (malformed decks whose equations fail to assemble): the symbols of the
deck without its equations, the equation text and the reference's message.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

DECKS = "/root/reference/proj/tests/decks"
RUNS = {"dam_break_2d": 10, "hot_start_demo": 10, "cahn_hilliard_patch": 10,
        "particle_damper": 10, "sampling_1k": 1, "sfm_agent": 10}
SAVE = (1, 10)
ERRORS = ["02_unknown_symbol", "06_unknown_function", "07_wrong_arity", "08_bad_kernel",
          "10_constant_lhs"]
SEED = 7
# equations that assemble but fail when solved (appended to dam_break_2d's list)
RUNTIME_ERRORS = [("lhs_shape", "v=rho"), ("add_shape", "p=v+rho"), ("nan_audit", "p=rho/(rho-rho)"),
                  ("var_shape", "dt=v"), ("dot_shape", "p=dot(v,rho)"),
                  ("join", "v=v|rho"), ("euler_dt", "p=euler(p,p,v)"),
                  ("builtin", "p=max(v,g|g)"), ("var_nan", "dt=dt/0")]


def state(rc, fields):
    return {name: rc.get(name) for name, _ in fields}


def deck_case(name, out):
    items = ref.deck_items(os.path.join(DECKS, name + ".yaml"))
    rc = ref.AssembledCase(items, seed=SEED)
    fields = rc.symbols(2)
    seed, counters = rc.rand_state()
    meta = {"domain": rc.domain, "n": rc.n, "seed": seed,
            "constants": [(n, v.tolist()) for n, v in rc.symbols(0)],
            "variables": [(n, v.tolist()) for n, v in rc.symbols(1)],
            "fields": [(n, list(s)) for n, s in fields],
            "equations": rc.equations(), "steps": [s for s in SAVE if s <= RUNS[name]]}
    out[f"{name}_meta"] = np.array(json.dumps(meta))
    for f, v in state(rc, fields).items():
        out[f"{name}_s0_{f}"] = v
    out[f"{name}_s0_rand"] = counters
    for s in range(1, RUNS[name] + 1):
        rc.solve_step(1)
        if s in meta["steps"]:
            for f, v in state(rc, fields).items():
                out[f"{name}_s{s}_{f}"] = v
            out[f"{name}_s{s}_active"] = rc.active()
            out[f"{name}_s{s}_vars"] = np.array(json.dumps(
                [(n, rc.get_variable(n).tolist()) for n, _ in meta["variables"]]))
    return meta


def error_case(name, out):
    items = ref.deck_items(os.path.join(DECKS, "malformed", name + ".yaml"))
    eqs = [it for it in items if it[0] == "equation"]
    try:
        ref.AssembledCase(items, seed=SEED)
        raise SystemExit(f"{name}: expected an assembly error")
    except ref.RefError as e:
        msg = str(e)
    base = ref.AssembledCase([it for it in items if it[0] != "equation"] +
                             [("equation", "noop", "dt=dt")], seed=SEED)
    meta = {"domain": base.domain, "n": base.n,
            "constants": [(n, v.tolist()) for n, v in base.symbols(0)],
            "variables": [(n, v.tolist()) for n, v in base.symbols(1)],
            "fields": [(n, list(s)) for n, s in base.symbols(2)],
            "equations": [(n, e) for _, n, e in eqs], "message": msg}
    out[f"err_{name}_meta"] = np.array(json.dumps(meta))
    out[f"err_{name}_r"] = base.get("r")
    for f, _ in meta["fields"]:
        out[f"err_{name}_f_{f}"] = base.get(f)


def runtime_error_case(key, text, out):
    items = ref.deck_items(os.path.join(DECKS, "dam_break_2d.yaml")) + [("equation", key, text)]
    rc = ref.AssembledCase(items, seed=SEED)
    try:
        rc.solve_step(1)
        raise SystemExit(f"{key}: expected a solve error")
    except ref.RefError as e:
        out[f"rt_{key}"] = np.array(json.dumps({"text": text, "message": str(e)}))
        return str(e)


def main():
    out = {}
    index = {"decks": [], "errors": []}
    for name in RUNS:
        meta = deck_case(name, out)
        index["decks"].append(name)
        print(name, meta["n"], "particles,", len(meta["equations"]), "equations")
    for name in ERRORS:
        error_case(name, out)
        index["errors"].append(name)
        print(name, json.loads(str(out[f"err_{name}_meta"]))["message"])
    index["runtime_errors"] = []
    for key, text in RUNTIME_ERRORS:
        print(key, runtime_error_case(key, text, out))
        index["runtime_errors"].append(key)
    out["index"] = np.array(json.dumps(index))
    np.savez_compressed(os.path.join(HERE, "decks.npz"), **out)


if __name__ == "__main__":
    main()
