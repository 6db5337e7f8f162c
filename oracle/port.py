"""TEST INFRASTRUCTURE: ctypes wrapper of oracle/nau_oracle.c (the C restatement).

Arrays are numpy, SoA component-major: a field with C components over n
particles is a (C, n) float64 array. Integer tables are int32.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libnau_oracle.so")

PERIODIC, SYMMETRIC, CUTOFF = 0, 1, 2
SPH_S, SPH_D00, SPH_G11, SPH_L0, SPH_A, DEM_HERTZ, DEM_BOUNDARY, GRAVITY, DEM_LSD, SFM = range(10)
K_WENDLAND, K_CUBIC = 0, 1


class NorDomain(C.Structure):
    _fields_ = [("dim", C.c_int), ("cells", C.c_int * 3), ("lo", C.c_double * 3),
                ("hi", C.c_double * 3), ("ext", C.c_double * 3), ("cs", C.c_double * 3),
                ("kind", C.c_int * 3)]


class NorOperand(C.Structure):
    _fields_ = [("field", C.c_void_p), ("value", C.c_double * 9), ("rows", C.c_int),
                ("cols", C.c_int)]


class NorPS(C.Structure):
    _fields_ = [("dom", NorDomain), ("n", C.c_int), ("pos", C.c_void_p), ("active", C.c_void_p),
                ("cell_of", C.c_void_p), ("cell_start", C.c_void_p), ("cell_count", C.c_void_p),
                ("sorted", C.c_void_p), ("warnings", C.c_long)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.run(["make", "-s", "-C", HERE, os.path.join(HERE, "_build", "libnau_oracle.so")],
                           check=True)
        L = C.CDLL(LIB_PATH)
        L.nor_domain_init.argtypes = [C.POINTER(NorDomain), C.c_int, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]
        L.nor_ncells.restype = C.c_long
        L.nor_cell_index.argtypes = [C.POINTER(NorDomain), C.c_int, C.c_double]
        L.nor_build_cells.restype = C.c_long
        L.nor_build_cells.argtypes = [C.POINTER(NorDomain), C.c_int] + [C.c_void_p] * 6
        L.nor_boundary_shift.restype = C.c_long
        L.nor_boundary_shift.argtypes = [C.POINTER(NorDomain), C.c_int, C.c_void_p, C.c_void_p]
        L.nor_neighbor_counts.argtypes = [C.POINTER(NorPS), C.c_double, C.c_void_p]
        L.nor_kernel_value.restype = C.c_double
        L.nor_kernel_value.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double]
        L.nor_kernel_dq.restype = C.c_double
        L.nor_kernel_dq.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double]
        L.nor_interact.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(NorPS),
                                   C.POINTER(NorOperand), C.c_int, C.c_void_p, C.c_int,
                                   C.POINTER(C.c_long)]
        L.nor_euler.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                C.c_void_p]
        L.nor_uniform_draws.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_double, C.c_double,
                                        C.c_void_p]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class Domain:
    """Mirror of include/nauticle/domain.hpp:19-49 (integer cell counts x cell size)."""

    def __init__(self, dim, min_cells, max_cells, cell_size, kinds):
        self.dim = dim
        self.min_cells = [int(v) for v in list(min_cells) + [0] * (3 - len(min_cells))]
        self.max_cells = [int(v) for v in list(max_cells) + [1] * (3 - len(max_cells))]
        self.cell_size = [float(v) for v in list(cell_size) + [1.0] * (3 - len(cell_size))]
        self.kinds = [int(v) for v in list(kinds) + [CUTOFF] * (3 - len(kinds))]
        self.c = NorDomain()
        mn = np.array(self.min_cells, np.int32)
        mx = np.array(self.max_cells, np.int32)
        cs = np.array(self.cell_size, np.float64)
        kd = np.array(self.kinds, np.int32)
        lib().nor_domain_init(C.byref(self.c), dim, _p(mn), _p(mx), _p(cs), _p(kd))

    @property
    def cells(self):
        return list(self.c.cells)

    @property
    def lo(self):
        return list(self.c.lo)

    @property
    def hi(self):
        return list(self.c.hi)

    @property
    def ncells(self):
        return int(lib().nor_ncells(C.byref(self.c)))


class OracleError(RuntimeError):
    def __init__(self, msg, particle):
        super().__init__(msg)
        self.particle = particle


class ParticleSystem:
    """CPU mirror of ParticleSystem (include/nauticle/particle_system.hpp:23-153)."""

    def __init__(self, dom: Domain, pos: np.ndarray, active=None):
        self.dom = dom
        self.pos = np.ascontiguousarray(pos, dtype=np.float64).copy()
        self.n = self.pos.shape[1]
        self.active = (np.ones(self.n, np.uint8) if active is None
                       else np.ascontiguousarray(active, dtype=np.uint8).copy())
        self.warnings = 0
        self.tables = None

    def boundary_shift(self):
        self.warnings += int(lib().nor_boundary_shift(C.byref(self.dom.c), self.n, _p(self.pos),
                                                      _p(self.active)))
        self.tables = None

    def build_cells(self):
        nc = self.dom.ncells
        cell_of = np.empty(self.n, np.int32)
        start = np.empty(nc, np.int32)
        count = np.empty(nc, np.int32)
        srt = np.empty(max(1, self.n), np.int32)
        bad = lib().nor_build_cells(C.byref(self.dom.c), self.n, _p(self.pos), _p(self.active),
                                    _p(cell_of), _p(start), _p(count), _p(srt))
        if bad:
            raise OracleError("particle outside the domain on a cut-off axis", bad - 1)
        nact = int(count.sum())
        self.tables = (cell_of, start, count, srt[:nact].copy() if nact else srt[:0].copy())
        self._srt_full = srt
        return self.tables

    def _ps(self):
        if self.tables is None:
            self.build_cells()
        cell_of, start, count, _ = self.tables
        ps = NorPS()
        ps.dom = self.dom.c
        ps.n = self.n
        ps.pos = _p(self.pos).value
        ps.active = _p(self.active).value
        ps.cell_of = _p(cell_of).value
        ps.cell_start = _p(start).value
        ps.cell_count = _p(count).value
        ps.sorted = _p(self._srt_full).value
        ps.warnings = 0
        return ps

    def neighbor_counts(self, radius):
        ps = self._ps()
        out = np.zeros(self.n, np.int32)
        lib().nor_neighbor_counts(C.byref(ps), float(radius), _p(out))
        return out

    def interact(self, op, operands, out_shape, kfamily=K_WENDLAND, kdim=None, init=None):
        """operands: list of (n,)/(C,n) arrays or python scalars / small tuples (uniform).

        out_shape = (rows, cols). Inactive particles keep `init` (default 0).
        """
        ps = self._ps()
        keep = []
        arr = (NorOperand * len(operands))()
        for k, o in enumerate(operands):
            rows, cols = 1, 1
            if isinstance(o, np.ndarray) and o.ndim >= 1 and o.shape[-1] == self.n:
                a = np.ascontiguousarray(np.atleast_2d(o), dtype=np.float64)
                keep.append(a)
                arr[k].field = _p(a).value
                rows = a.shape[0]
            else:
                v = np.atleast_1d(np.asarray(o, dtype=np.float64)).ravel()
                for c, x in enumerate(v):
                    arr[k].value[c] = x
                rows = v.size
            arr[k].rows, arr[k].cols = rows, cols
        comps = out_shape[0] * out_shape[1]
        out = (np.zeros((comps, self.n)) if init is None
               else np.ascontiguousarray(init, dtype=np.float64).reshape(comps, self.n).copy())
        bad = C.c_long(-1)
        rc = lib().nor_interact(op, kfamily, kdim if kdim else self.dom.dim, C.byref(ps), arr,
                                len(operands), _p(out), comps, C.byref(bad))
        self.warnings += ps.warnings
        if rc:
            raise OracleError(f"operator {op} failed", bad.value)
        return out


def kernel_value(family, kdim, h, d):
    return lib().nor_kernel_value(family, kdim, h, d)


def kernel_dq(family, kdim, h, q):
    return lib().nor_kernel_dq(family, kdim, h, q)


def uniform_draws(seed, n, ndraws, a=0.0, b=1.0):
    out = np.empty((ndraws, n), np.float64)
    lib().nor_uniform_draws(C.c_uint64(seed), n, ndraws, a, b, _p(out))
    return out


def euler(x, xdot, dt, active):
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.shape[-1]
    comps = x.size // n
    out = np.empty_like(x)
    lib().nor_euler(n, comps, _p(np.ascontiguousarray(active, np.uint8)), _p(x),
                    _p(np.ascontiguousarray(xdot, dtype=np.float64)), dt, _p(out))
    return out
