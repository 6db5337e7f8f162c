"""Golden fixtures for the device SFL evaluator (nau_eval).

Run in the build container (needs oracle/_ref/libnauticle_ref.so):

    make -C oracle && python tests/golden/make_vm_golden.py

Every expression is evaluated by the reference's own parser and AST evaluator
(sfl/parser.cpp, sfl/ast.cpp, tensor.cpp via oracle/ref_harness.cpp nref_eval)
over random fields of every Tensor shape class; the outputs and the reference's
error messages for shape errors are stored in tests/golden/vm_cases.npz.
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

N = 1500

EXPRESSIONS = [
    "s+t", "s-t*c", "u+w", "u-w*s", "s*u", "u*s", "M*u", "M*N", "N*M*u", "u/s", "M/c",
    "u/w", "-u", "-(s*t)", "s-(-t)", "-2^2*s", "s^2", "s^t", "u^2", "2^u", "abs(M)^t",
    "s<t", "s>t", "s<=t", "s>=t", "s==s", "t!=t", "(s>0.7)*u", "t|s", "t|s|c",
    "(t|s|c)+u", "exp(t)", "log(s)", "sin(t)*cos(s)", "tan(t)", "sqrt(s)", "abs(t)",
    "floor(t*3)", "sgn(t)", "norm(u)", "norm(M)", "min(s,t)", "max(u,t)", "min(t,u)",
    "max(M,N)", "dot(u,w)", "dot(M,N)", "dot(u,cv)", "c*u+cv", "M*(u+w)-N*u",
]

# rand(a, b): evaluated on a fresh case each (zero draw counters), the last one twice
# on the same case (the counters persist: the second draw differs)
RAND_EXPRESSIONS = ["rand(0,1)", "s*rand(-1,1)+rand(t-1,t+1)", "rand(0,s)|t"]

ERRORS = ["u+s", "s-u", "u*w", "s/u", "u^M", "u<s", "u|s", "(t|s|c)|s", "dot(u,s)", "M*w|s",
          "rand(u,s)"]


def make_case(seed=4242):
    rng = np.random.default_rng(seed)
    pos = rng.random((3, N))
    fields = {
        "s": rng.uniform(0.5, 2.0, (1, N)),
        "t": rng.uniform(-1.0, 1.0, (1, N)),
        "u": rng.uniform(-1.0, 1.0, (3, N)),
        "w": rng.uniform(0.2, 1.0, (3, N)) * np.where(rng.random((3, N)) < 0.5, -1.0, 1.0),
        "M": rng.uniform(-1.0, 1.0, (9, N)),
        "N": rng.uniform(-1.0, 1.0, (9, N)),
    }
    shapes = {"s": (1, 1), "t": (1, 1), "u": (3, 1), "w": (3, 1), "M": (3, 3), "N": (3, 3)}
    consts = {"c": np.array([[2.5]]), "cv": np.array([[1.0], [-2.0], [0.5]])}
    return pos, fields, shapes, consts


def main():
    pos, fields, shapes, consts = make_case()
    rc = ref.RefCase(3, [0, 0, 0], [2, 2, 2], [0.5, 0.5, 0.5], [2, 2, 2], pos)
    for k, v in fields.items():
        rows, cols = shapes[k]
        rc.field(k, v, rows=rows, cols=cols)
    for k, v in consts.items():
        rc.constant(k, v)
    out = {"pos": pos, "meta": np.array(json.dumps({
        "shapes": shapes, "consts": {k: v.tolist() for k, v in consts.items()},
        "expressions": EXPRESSIONS, "errors": ERRORS, "rand": RAND_EXPRESSIONS,
        "rand_seed": 7}))}
    for k, v in fields.items():
        out["f_" + k] = v
    import sfl_mini
    for idx, e in enumerate(EXPRESSIONS):
        # the output size from the lowering's host interpreter; the reference must agree
        sym = {k: ("field", j) for j, k in enumerate(fields)}
        sym.update({k: ("const", v) for k, v in consts.items()})
        prog, res = sfl_mini.lower(e, sym)
        fl = {j: (shapes[k][0], shapes[k][1], fields[k]) for j, k in enumerate(fields)}
        comps = sfl_mini.run_numpy(prog, res, fl, N).shape[0]
        out[f"e{idx}"] = rc.eval(e, comps)
    for idx, e in enumerate(RAND_EXPRESSIONS):
        rr = ref.RefCase(3, [0, 0, 0], [2, 2, 2], [0.5, 0.5, 0.5], [2, 2, 2], pos, seed=7)
        for k, v in fields.items():
            rows, cols = shapes[k]
            rr.field(k, v, rows=rows, cols=cols)
        comps = 2 if "|" in e else 1
        out[f"r{idx}"] = rr.eval(e, comps)
        if idx == len(RAND_EXPRESSIONS) - 1:
            out[f"r{idx}_again"] = rr.eval(e, comps)
    msgs = []
    for e in ERRORS:
        try:
            rc.eval(e, 9)
            msgs.append("")
        except ref.RefError as err:
            msgs.append(str(err))
    out["error_messages"] = np.array(json.dumps(msgs))
    np.savez_compressed(os.path.join(HERE, "vm_cases.npz"), **out)
    print("wrote", len(EXPRESSIONS), "expressions,", len(ERRORS), "error cases")
    for e, m in zip(ERRORS, msgs):
        print(f"  {e!r}: {m}")


if __name__ == "__main__":
    main()
