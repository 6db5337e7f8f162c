"""TEST INFRASTRUCTURE: ctypes wrapper of oracle/_ref/libnauticle_ref.so.

That library is the reference's own C++ (/root/reference/proj/src) compiled
unmodified against oracle/shim/ by oracle/Makefile, plus oracle/ref_harness.cpp
which drives it through its public API. It exists only where the build ran
(this container, or a GPU box that received the prebuilt .so).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libnauticle_ref.so")
UNIT_PATH = os.path.join(HERE, "_ref", "ref_unit")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        vp, i, d, cp = C.c_void_p, C.c_int, C.c_double, C.c_char_p
        L.nref_last_error.restype = cp
        L.nref_uniform_draws.argtypes = [C.c_uint64, i, i, d, d, vp]
        L.nref_create.restype = vp
        L.nref_create.argtypes = [i, vp, vp, vp, vp, i, vp, C.c_uint64]
        L.nref_destroy.argtypes = [vp]
        for f in (L.nref_add_constant, L.nref_add_variable, L.nref_add_field):
            f.argtypes = [vp, cp, i, i, vp]
        L.nref_get_field.argtypes = [vp, cp, vp, C.POINTER(i), C.POINTER(i)]
        L.nref_add_equation.argtypes = [vp, cp, cp]
        L.nref_solve_step.argtypes = [vp, i]
        L.nref_write_vtk.argtypes = [vp, cp, i, i, d, d]
        L.nref_eval.argtypes = [vp, cp, i, i, i, vp, C.POINTER(i)]
        L.nref_eval_law.argtypes = [vp, cp, i, C.POINTER(cp), i, i, i, i, vp, C.POINTER(i)]
        L.nref_boundary_shift.argtypes = [vp]
        L.nref_build_cells.argtypes = [vp]
        L.nref_rebuild_count.restype = C.c_long
        L.nref_rebuild_count.argtypes = [vp]
        L.nref_warning_count.restype = C.c_long
        L.nref_warning_count.argtypes = [vp]
        L.nref_active.argtypes = [vp, vp]
        L.nref_cell_tables.argtypes = [vp, vp, vp, vp, vp]
        L.nref_neighbor_counts.argtypes = [vp, d, vp]
        L.nref_kernel_value.restype = d
        L.nref_kernel_value.argtypes = [cp, d, d]
        L.nref_case_ptr.restype = vp
        L.nref_case_ptr.argtypes = [vp]
        L.nref_assemble.restype = vp
        L.nref_assemble.argtypes = [C.POINTER(cp), C.POINTER(cp), C.POINTER(cp), i, C.c_uint64]
        L.nref_domain.argtypes = [vp, C.POINTER(i), vp, vp, vp, vp]
        L.nref_symbol.argtypes = [vp, i, i, cp, i, C.POINTER(i), C.POINTER(i), vp]
        L.nref_equation.argtypes = [vp, i, cp, i, cp, i]
        L.nref_rand_counters.argtypes = [vp, C.POINTER(C.c_uint64), vp]
        L.nref_get_variable.argtypes = [vp, cp, vp, C.POINTER(i), C.POINTER(i)]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class RefError(RuntimeError):
    pass


def _check(rc):
    if rc != 0:
        raise RefError(lib().nref_last_error().decode())


def uniform_draws(seed, n, ndraws, a=0.0, b=1.0):
    out = np.empty((ndraws, n), np.float64)
    lib().nref_uniform_draws(C.c_uint64(seed), n, ndraws, a, b, _p(out))
    return out


def kernel_value(keyword: str, h: float, d: float) -> float:
    return lib().nref_kernel_value(keyword.encode(), h, d)


class RefCase:
    """A reference Case assembled the way tests/helpers.hpp:26-80 (CaseBuilder) does."""

    def __init__(self, dim, min_cells, max_cells, cell_size, kinds, pos, seed=0):
        self.dim = dim
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        self.n = pos.shape[1]
        pad = lambda v, f: np.array(list(v) + [f] * (3 - len(v)))
        self._keep = [pad(min_cells, 0).astype(np.int32), pad(max_cells, 1).astype(np.int32),
                      pad(cell_size, 1.0).astype(np.float64), pad(kinds, 2).astype(np.int32)]
        h = lib().nref_create(dim, *[_p(a) for a in self._keep], self.n, _p(pos), C.c_uint64(seed))
        if not h:
            raise RefError(lib().nref_last_error().decode())
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().nref_destroy(self.h)
            self.h = None

    @staticmethod
    def _tensor(v):
        a = np.atleast_2d(np.asarray(v, dtype=np.float64))
        if a.shape[0] == 1 and np.ndim(v) == 1:
            a = a.T  # a python vector is a column
        return a

    def constant(self, name, value):
        a = self._tensor(value)
        _check(lib().nref_add_constant(self.h, name.encode(), a.shape[0], a.shape[1],
                                       _p(np.asfortranarray(a).ravel(order="F").copy())))
        return self

    def variable(self, name, value):
        a = self._tensor(value)
        _check(lib().nref_add_variable(self.h, name.encode(), a.shape[0], a.shape[1],
                                       _p(np.asfortranarray(a).ravel(order="F").copy())))
        return self

    def field(self, name, soa, rows=None, cols=1):
        soa = np.ascontiguousarray(np.atleast_2d(np.asarray(soa, dtype=np.float64)))
        rows = rows or soa.shape[0] // cols
        _check(lib().nref_add_field(self.h, name.encode(), rows, cols, _p(soa)))
        return self

    def get(self, name):
        r, c = C.c_int(0), C.c_int(0)
        k = lib().nref_get_field(self.h, name.encode(), None, C.byref(r), C.byref(c))
        if k < 0:
            raise RefError(lib().nref_last_error().decode())
        out = np.empty((k, self.n), np.float64)
        lib().nref_get_field(self.h, name.encode(), _p(out), C.byref(r), C.byref(c))
        return out

    def equation(self, name, text):
        _check(lib().nref_add_equation(self.h, name.encode(), text.encode()))
        return self

    def case_ptr(self):
        """The reference Case object (for integration/gpu_case.cpp's tests)."""
        return lib().nref_case_ptr(self.h)

    def write_vtk(self, path, binary, frame_index=0, time=0.0, simulated_time=0.0):
        """The reference's make_frame + write_vtk (io/vtk.cpp:193-304)."""
        _check(lib().nref_write_vtk(self.h, str(path).encode(), int(binary), int(frame_index),
                                    float(time), float(simulated_time)))

    def solve_step(self, threads=1):
        _check(lib().nref_solve_step(self.h, threads))

    def eval(self, expr, comps, i0=0, count=None, threads=1, init=0.0):
        count = self.n if count is None else count
        out = np.full((comps, count), init, np.float64)
        nc = C.c_int(0)
        _check(lib().nref_eval(self.h, expr.encode(), i0, count, threads, _p(out), C.byref(nc)))
        return out

    def eval_law(self, op, operands, comps, kdim=None, i0=0, count=None, threads=1):
        count = self.n if count is None else count
        out = np.zeros((comps, count), np.float64)
        arr = (C.c_char_p * len(operands))(*[o.encode() for o in operands])
        nc = C.c_int(0)
        _check(lib().nref_eval_law(self.h, op.encode(), kdim or self.dim, arr, len(operands), i0,
                                   count, threads, _p(out), C.byref(nc)))
        return out

    def boundary_shift(self):
        _check(lib().nref_boundary_shift(self.h))

    def build_cells(self):
        _check(lib().nref_build_cells(self.h))

    @property
    def rebuild_count(self):
        return lib().nref_rebuild_count(self.h)

    @property
    def warning_count(self):
        return lib().nref_warning_count(self.h)

    def active(self):
        out = np.empty(self.n, np.uint8)
        lib().nref_active(self.h, _p(out))
        return out

    def cell_tables(self, ncells):
        cell_of = np.empty(self.n, np.int32)
        start = np.empty(ncells, np.int32)
        count = np.empty(ncells, np.int32)
        srt = np.empty(max(1, self.n), np.int32)
        rc = lib().nref_cell_tables(self.h, _p(cell_of), _p(start), _p(count), _p(srt))
        if rc < 0:
            raise RefError(lib().nref_last_error().decode())
        return cell_of, start, count, srt[: int(count.sum())].copy()

    def neighbor_counts(self, radius):
        out = np.empty(self.n, np.int32)
        _check(lib().nref_neighbor_counts(self.h, radius, _p(out)))
        return out


def _cstrs(items):
    arr = (C.c_char_p * max(1, len(items)))(*[x.encode() for x in items])
    return arr


class AssembledCase(RefCase):
    """A whole deck through the reference's own assemble_case (src/assemble.cpp): the
    document bindings come from the deck file (parsed by the caller; the reference's
    yaml-cpp reader is the one source left out of oracle/_ref)."""

    def __init__(self, items, seed=0):
        secs, names, exprs = zip(*items) if items else ((), (), ())
        keep = [_cstrs(list(secs)), _cstrs(list(names)), _cstrs(list(exprs))]
        h = lib().nref_assemble(keep[0], keep[1], keep[2], len(items), C.c_uint64(seed))
        if not h:
            raise RefError(lib().nref_last_error().decode())
        self.h = h
        dim = C.c_int(0)
        mn, mx = np.zeros(3, np.int32), np.zeros(3, np.int32)
        cs, kd = np.zeros(3), np.zeros(3, np.int32)
        self.n = lib().nref_domain(h, C.byref(dim), _p(mn), _p(mx), _p(cs), _p(kd))
        self.dim = dim.value
        d = self.dim
        self.domain = {"dim": d, "min_cells": mn[:d].tolist(), "max_cells": mx[:d].tolist(),
                       "cell_size": cs[:d].tolist(), "kinds": kd[:d].tolist()}

    def symbols(self, kind):
        """kind 0 constants, 1 variables, 2 fields: [(name, value (rows, cols) or shape)]."""
        out = []
        name = C.create_string_buffer(256)
        r, c = C.c_int(0), C.c_int(0)
        cnt = lib().nref_symbol(self.h, kind, -1, name, 256, C.byref(r), C.byref(c), None)
        for k in range(cnt):
            v = np.zeros(9)
            lib().nref_symbol(self.h, kind, k, name, 256, C.byref(r), C.byref(c), _p(v))
            val = v[: r.value * c.value].reshape(c.value, r.value).T.copy()
            out.append((name.value.decode(), val if kind < 2 else (r.value, c.value)))
        return out

    def equations(self):
        nb, tb = C.create_string_buffer(256), C.create_string_buffer(4096)
        cnt = lib().nref_equation(self.h, -1, nb, 256, tb, 4096)
        out = []
        for k in range(cnt):
            lib().nref_equation(self.h, k, nb, 256, tb, 4096)
            out.append((nb.value.decode(), tb.value.decode()))
        return out

    def rand_state(self):
        seed = C.c_uint64(0)
        cnt = np.zeros(self.n, np.uint64)
        lib().nref_rand_counters(self.h, C.byref(seed), _p(cnt))
        return seed.value, cnt

    def get_variable(self, name):
        v = np.zeros(9)
        r, c = C.c_int(0), C.c_int(0)
        k = lib().nref_get_variable(self.h, name.encode(), _p(v), C.byref(r), C.byref(c))
        if k < 0:
            raise RefError(lib().nref_last_error().decode())
        return v[:k].reshape(c.value, r.value).T.copy()


def deck_items(path):
    """CaseDocument bindings of a deck file, in document order (the schema of
    io/case_file.cpp; scalars kept as the file's text)."""
    import yaml
    with open(path) as f:
        doc = yaml.load(f, Loader=yaml.BaseLoader)
    case = doc["simulation"]["case"]
    ws = case["workspace"]
    items = []
    for sec, key in (("constant", "constants"), ("variable", "variables"), ("field", "fields")):
        for b in ws.get(key, []) or []:
            (name, expr), = b.items()
            items.append((sec, name, expr))
    ps = ws["particle_system"]
    for k, v in ps["domain"].items():
        items.append(("domain", k, v))
    for k, v in ps["grid"].items():
        items.append(("grid", k, v))
    for b in case.get("equations", []) or []:
        (name, expr), = b.items()
        items.append(("equation", name, expr))
    for k, v in (doc["simulation"].get("parameter_space") or {}).items():
        items.append(("param", k, v))
    return items
