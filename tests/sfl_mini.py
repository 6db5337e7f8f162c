"""Test utility: lower SFL particle-wise expressions to nau_eval programs.

A small restatement of the reference's expression grammar (sfl/parser.cpp:40-110:
'|' < comparisons < + - < * / < unary minus < '^' (right-assoc), negated
literals folded) for the particle-wise subset the device evaluator covers
(sfl/ast.cpp:71-175; builtins parser.cpp:218-240). The reference's own parser
is host-side setup and stays out of scope; this lowering only
lets the tests state each program once, as text, and run it through both the
reference (oracle.ref.RefCase.eval) and nau_eval.

`run_numpy` interprets a program on the host with the reference's Tensor rules
(tensor.cpp) and the shim's storage-order reductions: the CPU-side check of the
program semantics (tests/test_vm_oracle.py pins it against the reference).
"""
from __future__ import annotations

import re

import numpy as np

# opcodes (include/nauticle_gpu.h NAU_VM_*)
OPS = ["LOAD_FIELD", "LOAD_CONST", "ADD", "SUB", "MUL", "DIV", "POW", "LT", "GT", "LE", "GE",
       "EQ", "NE", "NEG", "JOIN", "EXP", "LOG", "SIN", "COS", "TAN", "SQRT", "ABS", "FLOOR",
       "SGN", "NORM", "MIN", "MAX", "DOT", "RAND"]
OP = {name: k for k, name in enumerate(OPS)}
UNARY = {"exp", "log", "sin", "cos", "tan", "sqrt", "abs", "floor", "sgn", "norm"}
BINARY = {"min", "max", "dot", "rand"}
CMP = {"<": "LT", ">": "GT", "<=": "LE", ">=": "GE", "==": "EQ", "!=": "NE"}
TRANSCENDENTAL = {"exp", "log", "sin", "cos", "tan", "^"}

_TOK = re.compile(r"\s*(?:(\d+\.?\d*(?:[eE][+-]?\d+)?|\.\d+(?:[eE][+-]?\d+)?)|([A-Za-z_]\w*)|"
                  r"(<=|>=|==|!=|[-+*/^<>|(),]))")


def tokenize(text):
    pos, out = 0, []
    text = text.strip()
    while pos < len(text):
        m = _TOK.match(text, pos)
        if not m or m.end() == pos:
            raise SyntaxError(f"bad token at {pos} in {text!r}")
        num, ident, op = m.groups()
        out.append(("num", float(num)) if num else ("id", ident) if ident else ("op", op))
        pos = m.end()
    out.append(("end", None))
    return out


class _Parser:
    """AST: ('lit', v) | ('sym', name) | ('bin', op, a, b) | ('neg', a) | ('join', a, b) |
    ('call', name, [args])."""

    def __init__(self, text):
        self.t = tokenize(text)
        self.i = 0

    def peek(self):
        return self.t[self.i]

    def accept(self, op):
        if self.t[self.i] == ("op", op):
            self.i += 1
            return True
        return False

    def parse(self):
        node = self.vector()
        if self.peek()[0] != "end":
            raise SyntaxError(f"trailing input at token {self.i}")
        return node

    def vector(self):
        node = self.comparison()
        while self.accept("|"):
            node = ("join", node, self.comparison())
        return node

    def comparison(self):
        node = self.additive()
        while True:
            tok = self.peek()
            if tok[0] == "op" and tok[1] in CMP:
                self.i += 1
                node = ("bin", tok[1], node, self.additive())
            else:
                return node

    def additive(self):
        node = self.multiplicative()
        while True:
            if self.accept("+"):
                node = ("bin", "+", node, self.multiplicative())
            elif self.accept("-"):
                node = ("bin", "-", node, self.multiplicative())
            else:
                return node

    def multiplicative(self):
        node = self.unary()
        while True:
            if self.accept("*"):
                node = ("bin", "*", node, self.unary())
            elif self.accept("/"):
                node = ("bin", "/", node, self.unary())
            else:
                return node

    def unary(self):
        if self.accept("-"):
            a = self.unary()
            if a[0] == "lit":
                return ("lit", -a[1])
            return ("neg", a)
        return self.power()

    def power(self):
        node = self.primary()
        if self.accept("^"):
            return ("bin", "^", node, self.unary())
        return node

    def primary(self):
        kind, val = self.peek()
        self.i += 1
        if kind == "num":
            return ("lit", val)
        if kind == "op" and val == "(":
            node = self.vector()
            if not self.accept(")"):
                raise SyntaxError("expected ')'")
            return node
        if kind == "id":
            if self.accept("("):
                args = []
                if not self.accept(")"):
                    args.append(self.vector())
                    while self.accept(","):
                        args.append(self.vector())
                    if not self.accept(")"):
                        raise SyntaxError("expected ')' after arguments")
                return ("call", val, args)
            return ("sym", val)
        raise SyntaxError(f"expected a value, got {kind} {val!r}")


def parse(text):
    return _Parser(text).parse()


_BIN = {"+": "ADD", "-": "SUB", "*": "MUL", "/": "DIV", "^": "POW", **CMP}


def lower(text, symbols):
    """Lower `text` to a program: list of dicts (op, dst, a, b, field, rows, cols, imm).
    symbols: name -> ("field", field_id) | ("const", np.array (rows, cols)).
    Register of a node = its depth in the evaluation stack (<= 16). Returns
    (program, result_register)."""
    prog = []

    def emit(op, dst, a=0, b=0, field=-1, value=None):
        ins = {"op": OP[op], "dst": dst, "a": a, "b": b, "field": field, "rows": 1, "cols": 1,
               "imm": [0.0] * 9}
        if value is not None:
            v = np.atleast_2d(np.asarray(value, dtype=np.float64))
            ins["rows"], ins["cols"] = v.shape
            ins["imm"][: v.size] = list(v.ravel(order="F"))
        prog.append(ins)

    def go(node, r):
        if r >= 16:
            raise ValueError("expression too deep for 16 registers")
        kind = node[0]
        if kind == "lit":
            emit("LOAD_CONST", r, value=[[node[1]]])
        elif kind == "sym":
            s = symbols[node[1]]
            if s[0] == "field":
                emit("LOAD_FIELD", r, field=s[1])
            else:
                emit("LOAD_CONST", r, value=s[1])
        elif kind == "bin":
            go(node[2], r)
            go(node[3], r + 1)
            emit(_BIN[node[1]], r, r, r + 1)
        elif kind == "neg":
            go(node[1], r)
            emit("NEG", r, r)
        elif kind == "join":
            go(node[1], r)
            go(node[2], r + 1)
            emit("JOIN", r, r, r + 1)
        elif kind == "call":
            name, args = node[1], node[2]
            if name in UNARY and len(args) == 1:
                go(args[0], r)
                emit(name.upper(), r, r)
            elif name in BINARY and len(args) == 2:
                go(args[0], r)
                go(args[1], r + 1)
                emit(name.upper(), r, r, r + 1)
            else:
                raise ValueError(f"unsupported call {name}/{len(args)}")
        else:
            raise ValueError(kind)

    go(parse(text), 0)
    return prog, 0


def uses_transcendental(text):
    ast = parse(text)
    found = False

    def walk(n):
        nonlocal found
        if n[0] == "bin" and n[1] == "^":
            found = True
        if n[0] == "call" and n[1] in TRANSCENDENTAL:
            found = True
        for c in n[1:]:
            if isinstance(c, tuple):
                walk(c)
            elif isinstance(c, list):
                for x in c:
                    walk(x)
    walk(ast)
    return found


# ------------------------------------------------------- host interpreter ----
M64 = (1 << 64) - 1


def _mix(x):
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def rand_uniform(seed, counters, a, b):
    """RandomState::uniform (sfl/random_state.hpp) for particles 0..n-1; advances counters."""
    out = np.empty(len(counters))
    s0 = _mix(seed ^ 0x6E61757469636C65)
    for i in range(len(counters)):
        x = _mix(s0 ^ _mix(i + 0x9E3779B9) ^ int(counters[i]))
        counters[i] += 1
        u = float(x >> 11) * 2.0 ** -53
        out[i] = a[i] + u * (b[i] - a[i])
    return out


def run_numpy(prog, result, fields, n, seed=0, counters=None):
    counters = np.zeros(n, dtype=np.uint64) if counters is None else counters
    with np.errstate(all="ignore"):
        return _run_numpy(prog, result, fields, n, seed, counters)


def _run_numpy(prog, result, fields, n, seed, counters):
    """Evaluate a program for n particles on the host. fields: id -> (rows, cols, soa
    (rows*cols, n) column-major components). Returns (rows*cols, n)."""
    regs = {}
    for ins in prog:
        op = OPS[ins["op"]]
        d = ins["dst"]
        if op == "LOAD_FIELD":
            rows, cols, soa = fields[ins["field"]]
            regs[d] = (rows, cols, np.array(soa, dtype=np.float64).reshape(rows * cols, n))
            continue
        if op == "LOAD_CONST":
            rows, cols = ins["rows"], ins["cols"]
            v = np.array(ins["imm"][: rows * cols])[:, None] * np.ones((1, n))
            regs[d] = (rows, cols, v)
            continue
        ar, ac, a = regs[ins["a"]]
        if op in ("NEG",) or op.lower() in UNARY:
            f = {"NEG": np.negative, "EXP": np.exp, "LOG": np.log, "SIN": np.sin, "COS": np.cos,
                 "TAN": np.tan, "SQRT": np.sqrt, "ABS": np.abs, "FLOOR": np.floor,
                 "SGN": lambda x: np.where(x > 0, 1.0, np.where(x < 0, -1.0, 0.0))}
            if op == "NORM":
                s = a[0] * a[0]
                for c in range(1, ar * ac):
                    s = s + a[c] * a[c]
                regs[d] = (1, 1, np.sqrt(s)[None, :])
            else:
                regs[d] = (ar, ac, f[op](a))
            continue
        br, bc, b = regs[ins["b"]]
        if op in ("ADD", "SUB"):
            assert (ar, ac) == (br, bc), f"operator shapes {ar}x{ac} {br}x{bc}"
            regs[d] = (ar, ac, a + b if op == "ADD" else a - b)
        elif op == "MUL":
            if (ar, ac) == (1, 1):
                regs[d] = (br, bc, a[0] * b)
            elif (br, bc) == (1, 1):
                regs[d] = (ar, ac, b[0] * a)
            else:
                assert ac == br
                out = np.empty((ar * bc, n))
                for r in range(ar):
                    for c in range(bc):
                        s = a[r] * b[c * br]
                        for q in range(1, ac):
                            s = s + a[q * ar + r] * b[c * br + q]
                        out[c * ar + r] = s
                regs[d] = (ar, bc, out)
        elif op == "DIV":
            regs[d] = (ar, ac, a / b[0] if (br, bc) == (1, 1) else a / b)
        elif op in ("POW", "MIN", "MAX"):
            f = {"POW": np.power, "MIN": np.fmin, "MAX": np.fmax}[op]
            if (ar, ac) == (1, 1) and (br, bc) != (1, 1):
                regs[d] = (br, bc, f(np.broadcast_to(a[0], b.shape).copy(), b))
            elif (br, bc) == (1, 1) and (ar, ac) != (1, 1):
                regs[d] = (ar, ac, f(a, np.broadcast_to(b[0], a.shape).copy()))
            else:
                regs[d] = (ar, ac, f(a, b))
        elif op in ("LT", "GT", "LE", "GE", "EQ", "NE"):
            f = {"LT": np.less, "GT": np.greater, "LE": np.less_equal, "GE": np.greater_equal,
                 "EQ": np.equal, "NE": np.not_equal}[op]
            regs[d] = (1, 1, f(a[0], b[0]).astype(np.float64)[None, :])
        elif op == "JOIN":
            regs[d] = (ar + 1, 1, np.concatenate([a, b[:1]], axis=0))
        elif op == "RAND":
            regs[d] = (1, 1, rand_uniform(seed, counters, a[0], b[0])[None, :])
        elif op == "DOT":
            s = a[0] * b[0]
            for c in range(1, ar * ac):
                s = s + a[c] * b[c]
            regs[d] = (1, 1, s[None, :])
        else:
            raise ValueError(op)
    return regs[result][2]
