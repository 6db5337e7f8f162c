"""ctypes binding of libnau_b200.so (include/nauticle_gpu.h).

This is the Python face of the C-ABI that tests/, bench.py and smoke() drive.
It mirrors the reference's host-side vocabulary — Domain, particle fields,
interaction operators looked up by their SFL names (kOps[],
/root/reference/proj/src/interactions.cpp:259-269), euler, reductions — and
raises NauError with the reference's error kinds (include/nauticle/error.hpp).

There is no CPU fallback: importing works anywhere, but creating a Context
loads the CUDA library and fails loudly if it is missing or no GPU is present.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# NAU_LIB: an alternative build of the same library (tools/variants.sh experiments)
LIB_PATH = os.environ.get("NAU_LIB") or os.path.join(HERE, "libnau_b200.so")

PERIODIC, SYMMETRIC, CUTOFF = 0, 1, 2
OPS = {"sph_S": 0, "sph_D00": 1, "sph_G11": 2, "sph_L0": 3, "sph_A": 4, "dem_l": 5,
       "dem_boundary_force": 6, "nbody_gravity": 7, "dem_lsd": 8, "sfm": 9}
K_WENDLAND, K_CUBIC = 0, 1
MODE_EXACT, MODE_FAST = 0, 1
STATUS = {0: "ok", 1: "runtime error", 2: "runtime NaN", 3: "CUDA error", 4: "argument error",
          5: "communication error"}

# Every symbol include/nauticle_gpu.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = [
    "nau_find_interaction", "nau_decode_kernel", "nau_create", "nau_destroy", "nau_set_stream",
    "nau_get_stream", "nau_set_domain", "nau_set_particles", "nau_particle_count",
    "nau_active_count", "nau_get_active", "nau_alloc_field", "nau_free_field", "nau_upload",
    "nau_download", "nau_fill", "nau_copy_field", "nau_field_device_ptr", "nau_boundary_shift",
    "nau_build_cells", "nau_cells_dirty", "nau_rebuild_count", "nau_warning_count", "nau_ncells",
    "nau_cell_tables", "nau_neighbor_counts", "nau_interact", "nau_interact_g11_l0", "nau_euler", "nau_symplectic_step",
    "nau_wcsph_step", "nau_reduce", "nau_sync", "nau_last_error", "nau_profile_enable",
    "nau_profile_ms", "nau_launch_count", "nau_wcsph_path", "nau_list_stats", "nau_fp64_peak_tflops", "nau_set_mode", "nau_get_mode",
    "nau_row_width", "nau_select", "nau_pack_rows", "nau_load_rows", "nau_dem_step",
    "nau_leapfrog_step", "nau_pack_sources", "nau_gravity_sources", "nau_gravity_sources_part", "nau_set_neighbor_lists",
    "nau_upload_async", "nau_download_async", "nau_io_fence", "nau_io_join", "nau_eval",
    "nau_set_random_state", "nau_get_random_counters", "nau_comm_unique_id", "nau_comm_init",
    "nau_comm_destroy", "nau_slab_config", "nau_migrate", "nau_halo_exchange", "nau_comm_swap",
    "nau_write_vtk", "nau_vtk_read", "nau_vtk_free", "nau_vtk_last_error", "nau_vtk_points",
    "nau_vtk_array_count", "nau_vtk_array", "nau_vtk_strings", "nau_vtk_rand_counters",
    "nau_allreduce", "nau_comm_size", "nau_field_shape", "nau_case_create", "nau_case_destroy",
    "nau_case_constant", "nau_case_variable", "nau_case_set_variable", "nau_case_get_variable",
    "nau_case_field", "nau_case_equation", "nau_case_equation_count", "nau_case_solve_equation",
    "nau_case_solve_step", "nau_case_last_error", "nau_wcsph_pass", "nau_select_x", "nau_reserve",
    "nau_rebuild_rows", "nau_histogram_x", "nau_set_ghost_field", "nau_wcsph_pack_rho_p",
    "nau_wcsph_ghost_update", "nau_slab_bounds", "nau_slab_rebalance", "nau_pack_fields",
    "nau_unpack_fields", "nau_wcsph_ghost_payload", "nau_set_graphs",
]


class NauError(RuntimeError):
    def __init__(self, status, message, particle=-1):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.message = message
        self.particle = particle


class OpInfo(C.Structure):
    _fields_ = [("name", C.c_char_p), ("op", C.c_int), ("arity_min", C.c_int),
                ("arity_max", C.c_int), ("kernel_slot", C.c_int), ("radius_slot", C.c_int),
                ("finite_influence", C.c_int)]


class Operand(C.Structure):
    _fields_ = [("field_id", C.c_int), ("rows", C.c_int), ("cols", C.c_int),
                ("value", C.c_double * 9)]


class WcsphParams(C.Structure):
    _fields_ = [("kernel_family", C.c_int), ("kernel_dim", C.c_int), ("mass", C.c_double),
                ("radius", C.c_double), ("rho0", C.c_double), ("B", C.c_double),
                ("gamma", C.c_double), ("visc", C.c_double), ("dt", C.c_double),
                ("g", C.c_double * 3), ("f_rho", C.c_int), ("f_p", C.c_int), ("f_v", C.c_int),
                ("f_vdot", C.c_int), ("f_mask", C.c_int)]


class DemParams(C.Structure):
    _fields_ = [("law", C.c_int), ("f_v", C.c_int), ("f_vdot", C.c_int), ("f_R", C.c_int),
                ("f_m", C.c_int), ("R", C.c_double), ("m", C.c_double), ("P", C.c_double),
                ("Q", C.c_double), ("cf", C.c_double), ("search_radius", C.c_double),
                ("dt", C.c_double), ("g", C.c_double * 3)]


class VmInstr(C.Structure):
    """nau_vm_instr (include/nauticle_gpu.h): one instruction of a nau_eval program."""
    _fields_ = [("op", C.c_int), ("dst", C.c_int), ("a", C.c_int), ("b", C.c_int),
                ("field", C.c_int), ("rows", C.c_int), ("cols", C.c_int), ("imm", C.c_double * 9)]


class GravityParams(C.Structure):
    _fields_ = [("f_v", C.c_int), ("f_a", C.c_int), ("f_m", C.c_int), ("m", C.c_double),
                ("G", C.c_double), ("eps", C.c_double), ("dt", C.c_double)]


_lib = None


def load():
    """Load the CUDA library (raises if it was not built: no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i, d, l = C.c_void_p, C.c_int, C.c_double, C.c_long
    sig = {
        "nau_find_interaction": (i, [C.c_char_p, C.POINTER(OpInfo)]),
        "nau_decode_kernel": (i, [C.c_char_p, C.POINTER(i), C.POINTER(i)]),
        "nau_create": (i, [i, C.POINTER(vp)]),
        "nau_destroy": (None, [vp]),
        "nau_set_stream": (i, [vp, vp]),
        "nau_get_stream": (vp, [vp]),
        "nau_set_domain": (i, [vp, i, vp, vp, vp, vp]),
        "nau_set_particles": (i, [vp, l, vp]),
        "nau_particle_count": (l, [vp]),
        "nau_active_count": (l, [vp]),
        "nau_get_active": (i, [vp, vp]),
        "nau_alloc_field": (i, [vp, i, i, C.POINTER(i)]),
        "nau_free_field": (i, [vp, i]),
        "nau_upload": (i, [vp, i, vp, l]),
        "nau_download": (i, [vp, i, vp, l]),
        "nau_fill": (i, [vp, i, vp]),
        "nau_copy_field": (i, [vp, i, i]),
        "nau_field_device_ptr": (i, [vp, i, C.POINTER(vp)]),
        "nau_boundary_shift": (i, [vp]),
        "nau_build_cells": (i, [vp]),
        "nau_cells_dirty": (i, [vp]),
        "nau_rebuild_count": (l, [vp]),
        "nau_warning_count": (l, [vp]),
        "nau_ncells": (l, [vp]),
        "nau_cell_tables": (i, [vp, vp, vp, vp, vp]),
        "nau_neighbor_counts": (i, [vp, d, vp]),
        "nau_interact": (i, [vp, i, i, i, C.POINTER(Operand), i, i]),
        "nau_interact_g11_l0": (i, [vp, i, i, C.POINTER(Operand), i, i, i]),
        "nau_euler": (i, [vp, i, i, d, i]),
        "nau_symplectic_step": (i, [vp, i, i, i, d]),
        "nau_wcsph_step": (i, [vp, C.POINTER(WcsphParams)]),
        "nau_reduce": (i, [vp, i, i, vp]),
        "nau_sync": (i, [vp]),
        "nau_last_error": (C.c_char_p, [vp, C.POINTER(l)]),
        "nau_profile_enable": (i, [vp, i]),
        "nau_profile_ms": (d, [vp, i, C.POINTER(l)]),
        "nau_launch_count": (l, [vp]),
        "nau_wcsph_path": (i, [vp]),
        "nau_list_stats": (i, [vp, C.POINTER(d)]),
        "nau_fp64_peak_tflops": (d, [i]),
        "nau_set_mode": (i, [vp, i]),
        "nau_get_mode": (i, [vp]),
        "nau_row_width": (i, [vp]),
        "nau_select": (i, [vp, i, d, d, i, d, d, vp, C.POINTER(l)]),
        "nau_pack_rows": (i, [vp, vp, l, vp]),
        "nau_load_rows": (i, [vp, vp, l, i]),
        "nau_dem_step": (i, [vp, C.POINTER(DemParams)]),
        "nau_leapfrog_step": (i, [vp, C.POINTER(GravityParams)]),
        "nau_pack_sources": (i, [vp, i, d, vp]),
        "nau_gravity_sources": (i, [vp, vp, l, l, d, d, i]),
        "nau_gravity_sources_part": (i, [vp, vp, l, l, d, d, i, i]),
        "nau_set_neighbor_lists": (i, [vp, i]),
        "nau_upload_async": (i, [vp, i, vp, l]),
        "nau_download_async": (i, [vp, i, vp, l]),
        "nau_io_fence": (i, [vp]),
        "nau_io_join": (i, [vp]),
        "nau_eval": (i, [vp, C.POINTER(VmInstr), i, i, i]),
        "nau_set_random_state": (i, [vp, C.c_ulonglong, vp]),
        "nau_get_random_counters": (i, [vp, vp]),
        "nau_comm_unique_id": (i, [vp]),
        "nau_comm_init": (i, [vp, vp, i, i]),
        "nau_comm_destroy": (None, [vp]),
        "nau_slab_config": (i, [vp, i, vp, i, d, i, i]),
        "nau_slab_bounds": (i, [vp, vp]),
        "nau_slab_rebalance": (i, [vp, i]),
        "nau_migrate": (i, [vp]),
        "nau_halo_exchange": (i, [vp, vp, i]),
        "nau_pack_fields": (i, [vp, vp, l, vp, i, vp]),
        "nau_unpack_fields": (i, [vp, vp, l, vp, i, vp]),
        "nau_wcsph_ghost_payload": (i, [vp, C.POINTER(WcsphParams)]),
        "nau_set_graphs": (i, [vp, i]),
        "nau_comm_swap": (i, [vp, vp, l, vp, l, i, vp, vp, vp, vp]),
        "nau_write_vtk": (i, [vp, C.c_char_p, i, vp]),
        "nau_vtk_read": (i, [C.c_char_p, vp]),
        "nau_vtk_free": (None, [vp]),
        "nau_vtk_last_error": (C.c_char_p, []),
        "nau_vtk_points": (l, [vp, vp, vp, vp, vp]),
        "nau_vtk_array_count": (i, [vp]),
        "nau_vtk_array": (C.c_char_p, [vp, i, vp, vp, vp]),
        "nau_vtk_strings": (i, [vp, C.c_char_p, vp]),
        "nau_vtk_rand_counters": (l, [vp, vp]),
        "nau_allreduce": (i, [vp, vp, i, i]),
        "nau_comm_size": (i, [vp]),
        "nau_field_shape": (i, [vp, i, C.POINTER(i), C.POINTER(i)]),
        "nau_case_create": (i, [vp, C.POINTER(vp)]),
        "nau_case_destroy": (None, [vp]),
        "nau_case_constant": (i, [vp, C.c_char_p, i, i, vp]),
        "nau_case_variable": (i, [vp, C.c_char_p, i, i, vp]),
        "nau_case_set_variable": (i, [vp, C.c_char_p, i, i, vp]),
        "nau_case_get_variable": (i, [vp, C.c_char_p, vp, C.POINTER(i), C.POINTER(i)]),
        "nau_case_field": (i, [vp, C.c_char_p, i]),
        "nau_case_equation": (i, [vp, C.c_char_p, C.c_char_p]),
        "nau_case_equation_count": (i, [vp]),
        "nau_case_solve_equation": (i, [vp, i]),
        "nau_case_solve_step": (i, [vp]),
        "nau_case_last_error": (C.c_char_p, [vp, C.POINTER(l)]),
        "nau_wcsph_pass": (i, [vp, C.POINTER(WcsphParams), i]),
        "nau_select_x": (i, [vp, i, d, d, i, d, d, vp, C.POINTER(l)]),
        "nau_reserve": (i, [vp, l]),
        "nau_rebuild_rows": (i, [vp, vp, l, vp, l, i]),
        "nau_histogram_x": (i, [vp, i, d, d, i, i, d, d, vp]),
        "nau_set_ghost_field": (i, [vp, i]),
        "nau_wcsph_pack_rho_p": (i, [vp, C.POINTER(WcsphParams), vp, l, vp]),
        "nau_wcsph_ghost_update": (i, [vp, C.POINTER(WcsphParams), vp, l, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class FrameMeta(C.Structure):
    _fields_ = [("frame_index", C.c_int), ("time", C.c_double), ("domain_text", C.c_char_p),
                ("params_text", C.c_char_p), ("n_variables", C.c_int),
                ("variables", C.POINTER(C.c_char_p)), ("n_constants", C.c_int),
                ("constants", C.POINTER(C.c_char_p)), ("n_equations", C.c_int),
                ("equations", C.POINTER(C.c_char_p)), ("n_fields", C.c_int),
                ("field_ids", C.POINTER(C.c_int)), ("field_names", C.POINTER(C.c_char_p))]


def _strs(items):
    arr = (C.c_char_p * max(1, len(items)))(*[s.encode() for s in items])
    return len(items), arr


def read_vtk(path):
    """The reference's read_vtk (io/vtk.cpp:310-464) through the library: a dict with
    dim, frame, time, pos (dim x n), arrays {name: (rows, cols) SoA}, strings, rand_counters."""
    L = load()
    h = C.c_void_p()
    if L.nau_vtk_read(str(path).encode(), C.byref(h)) != 0:
        raise NauError(1, L.nau_vtk_last_error().decode())
    try:
        dim, fidx, t, pp = C.c_int(), C.c_int(), C.c_double(), C.POINTER(C.c_double)()
        n = L.nau_vtk_points(h, C.byref(dim), C.byref(fidx), C.byref(t), C.byref(pp))
        pos = np.ctypeslib.as_array(pp, (dim.value * n,)).reshape(dim.value, n).copy() if n else \
            np.zeros((dim.value, 0))
        arrays = {}
        for k in range(L.nau_vtk_array_count(h)):
            r, cc, sp = C.c_int(), C.c_int(), C.POINTER(C.c_double)()
            name = L.nau_vtk_array(h, k, C.byref(r), C.byref(cc), C.byref(sp)).decode()
            comps = r.value * cc.value
            arrays[name] = ((r.value, cc.value),
                            np.ctypeslib.as_array(sp, (comps * n,)).reshape(comps, n).copy())
        strings = {}
        for key in ("domain", "params", "field_shapes", "variables", "constants", "equations"):
            items = C.POINTER(C.c_char_p)()
            m = L.nau_vtk_strings(h, key.encode(), C.byref(items))
            if m:
                strings[key] = [items[q].decode() for q in range(m)]
        cp = C.POINTER(C.c_ulonglong)()
        m = L.nau_vtk_rand_counters(h, C.byref(cp))
        rc = np.ctypeslib.as_array(cp, (m,)).copy() if m else np.zeros(0, np.uint64)
        return {"dim": dim.value, "frame": fidx.value, "time": t.value, "pos": pos,
                "arrays": arrays, "strings": strings, "rand_counters": rc}
    finally:
        L.nau_vtk_free(h)


def find_interaction(name):
    """≙ find_interaction (interactions.cpp:273-277); returns the kOps[] row as a dict."""
    L = load()
    info = OpInfo()
    if L.nau_find_interaction(name.encode(), C.byref(info)) != 0:
        raise NauError(4, L.nau_last_error(None, None).decode())
    return {"name": info.name.decode(), "op": info.op, "arity_min": info.arity_min,
            "arity_max": info.arity_max, "kernel_slot": info.kernel_slot,
            "radius_slot": info.radius_slot, "finite_influence": bool(info.finite_influence)}


def decode_kernel(keyword):
    """≙ decode_kernel_keyword (kernel.cpp:20-35), plus the cubic-spline family Wc3D220."""
    L = load()
    fam, dim = C.c_int(0), C.c_int(0)
    if L.nau_decode_kernel(keyword.encode(), C.byref(fam), C.byref(dim)) != 0:
        raise NauError(4, L.nau_last_error(None, None).decode())
    return fam.value, dim.value


def fp64_peak_tflops(device=0):
    return load().nau_fp64_peak_tflops(device)


class Field:
    def __init__(self, ctx, fid, rows, cols):
        self.ctx, self.id, self.rows, self.cols = ctx, fid, rows, cols

    @property
    def comps(self):
        return self.rows * self.cols


class Context:
    """One GPU context: domain, particles (field 0 = r) and SoA fields on the device."""

    def __init__(self, device=0):
        self.L = load()
        h = C.c_void_p()
        st = self.L.nau_create(device, C.byref(h))
        if st != 0:
            raise NauError(st, self.L.nau_last_error(None, None).decode())
        self.h = h
        self.n = 0
        self.dim = 0
        self.fields = {}

    # ---- native slab exchange over NCCL (comm.cu) ----
    @staticmethod
    def comm_unique_id() -> bytes:
        """128-byte NCCL id (rank 0); ship it to the other ranks."""
        L = load()
        buf = (C.c_ubyte * 128)()
        if L.nau_comm_unique_id(buf) != 0:
            raise NauError(5, "NCCL unavailable")
        return bytes(buf)

    def comm_init(self, uid: bytes, nranks: int, rank: int):
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        self._check(self.L.nau_comm_init(self.h, buf, nranks, rank))

    def slab_config(self, axis, bounds, periodic, radius, gid="gid", flag="ghost"):
        """x-threshold slabs: bounds = nranks + 1 coordinates (nau_slab_config)."""
        b = np.ascontiguousarray(bounds, dtype=np.float64)
        self._slab_nb = len(b)
        self._check(self.L.nau_slab_config(self.h, axis, b.ctypes.data, int(periodic),
                                           float(radius), self._fid(gid), self._fid(flag)))

    def slab_bounds(self):
        out = np.zeros(self._slab_nb)
        self._check(self.L.nau_slab_bounds(self.h, out.ctypes.data))
        return out.tolist()

    def migrate(self):
        self._check(self.L.nau_migrate(self.h))
        self.n = self.L.nau_particle_count(self.h)

    def halo_exchange(self, fields):
        ids = np.ascontiguousarray([self._fid(f) for f in fields], dtype=np.int32)
        self._check(self.L.nau_halo_exchange(self.h, ids.ctypes.data, len(ids)))

    def slab_rebalance(self, nbins=4096):
        self._check(self.L.nau_slab_rebalance(self.h, nbins))
        self.n = self.L.nau_particle_count(self.h)

    def comm_swap(self, to_left, to_right):
        """Swap device row blocks (torch float64, rows x width) with the neighbours;
        returns (from_left, from_right) as torch device tensors (copies)."""
        import torch
        w = int(to_left.shape[1])
        fl, fr = C.c_void_p(), C.c_void_p()
        nl, nr = C.c_long(), C.c_long()
        self._check(self.L.nau_comm_swap(self.h, to_left.data_ptr(), to_left.shape[0],
                                         to_right.data_ptr(), to_right.shape[0], w,
                                         C.byref(fl), C.byref(nl), C.byref(fr), C.byref(nr)))
        self.sync()
        out = []
        for p, m in ((fl, nl.value), (fr, nr.value)):
            if m == 0:
                out.append(torch.empty((0, w), dtype=torch.float64, device=to_left.device))
                continue

            class _View:  # the library-owned receive buffer as a CUDA array
                __cuda_array_interface__ = {"shape": (m, w), "typestr": "<f8",
                                            "data": (p.value, False), "version": 2}
            out.append(torch.as_tensor(_View(), device=to_left.device).clone())
        return out[0], out[1]

    def close(self):
        for cs in getattr(self, "_cases", []):
            cs.close()  # executors free their temporaries in this context first
        if getattr(self, "h", None):
            self.L.nau_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != 0:
            bad = C.c_long(-1)
            msg = self.L.nau_last_error(self.h, C.byref(bad)).decode()
            raise NauError(st, msg, bad.value)

    # ---- setup ----
    def set_mode(self, fast: bool):
        """EXACT (reference order, bitwise) or FAST (warp per particle, tolerance)."""
        self._check(self.L.nau_set_mode(self.h, MODE_FAST if fast else MODE_EXACT))

    @property
    def fast(self):
        return self.L.nau_get_mode(self.h) == MODE_FAST

    def set_neighbor_lists(self, on):
        """Per-step neighbour lists (identical results, faster): False/0 off, True/1 on
        (paired lists for the FAST Wendland wcsph_step), 2 on with per-particle lists only."""
        self._check(self.L.nau_set_neighbor_lists(self.h, int(on)))

    def set_stream(self, stream_ptr):
        self._check(self.L.nau_set_stream(self.h, C.c_void_p(stream_ptr)))

    def set_domain(self, dim, min_cells, max_cells, cell_size, kinds):
        pad = lambda v, f, t: np.array(list(v) + [f] * (3 - len(v)), t)
        self._dom = (pad(min_cells, 0, np.int32), pad(max_cells, 1, np.int32),
                     pad(cell_size, 1.0, np.float64), pad(kinds, CUTOFF, np.int32))
        self._check(self.L.nau_set_domain(self.h, dim, *[_p(a) for a in self._dom]))
        self.dim = dim

    def set_particles(self, pos):
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        assert pos.shape[0] == self.dim
        self.n = pos.shape[1]
        self._check(self.L.nau_set_particles(self.h, self.n, _p(pos)))
        self.fields = {"r": Field(self, 0, self.dim, 1)}
        return self.fields["r"]

    def add_field(self, name, rows=1, cols=1, values=None):
        fid = C.c_int(-1)
        self._check(self.L.nau_alloc_field(self.h, rows, cols, C.byref(fid)))
        f = Field(self, fid.value, rows, cols)
        self.fields[name] = f
        if values is not None:
            a = np.asarray(values, dtype=np.float64)
            if a.ndim >= 1 and a.shape[-1] == self.n and a.size == rows * cols * self.n:
                self.upload(f, a)
            else:
                self.fill(f, a)
        return f

    def field(self, name):
        return self.fields[name]

    def _fid(self, f):
        if isinstance(f, Field):
            return f.id
        if isinstance(f, str):
            return self.fields[f].id
        return int(f)

    def _comps(self, f):
        f = self.fields[f] if isinstance(f, str) else f
        return f.comps

    def upload(self, f, values):
        a = np.ascontiguousarray(np.atleast_2d(np.asarray(values, dtype=np.float64)))
        if a.shape[-1] != self.n or a.shape[0] != self._comps(f):
            a = np.ascontiguousarray(a.reshape(self._comps(f), self.n))
        self._check(self.L.nau_upload(self.h, self._fid(f), _p(a), self.n))

    def upload_ptr(self, f, host_ptr):
        """Upload from a raw host pointer (e.g. a pinned torch tensor's data_ptr())."""
        self._check(self.L.nau_upload(self.h, self._fid(f), C.c_void_p(host_ptr), self.n))

    def download(self, f):
        out = np.empty((self._comps(f), self.n), np.float64)
        self._check(self.L.nau_download(self.h, self._fid(f), _p(out), self.n))
        return out

    def download_ptr(self, f, host_ptr):
        self._check(self.L.nau_download(self.h, self._fid(f), C.c_void_p(host_ptr), self.n))

    def upload_async(self, f, host_ptr):
        """Asynchronous upload from a pinned host buffer (complete at sync())."""
        self._check(self.L.nau_upload_async(self.h, self._fid(f), C.c_void_p(host_ptr), self.n))

    def download_async(self, f, host_ptr):
        """Asynchronous download into a pinned host buffer (valid after sync())."""
        self._check(self.L.nau_download_async(self.h, self._fid(f), C.c_void_p(host_ptr), self.n))

    def eval_program(self, program, result, out):
        """≙ one particle-wise SFL equation `out = <program>` (nau_eval). `program` is a
        list of dicts with keys op, dst, a, b, field, rows, cols, imm (nau_vm_instr)."""
        arr = (VmInstr * len(program))()
        for k, ins in enumerate(program):
            arr[k].op, arr[k].dst, arr[k].a, arr[k].b = ins["op"], ins["dst"], ins["a"], ins["b"]
            arr[k].field, arr[k].rows, arr[k].cols = ins["field"], ins["rows"], ins["cols"]
            for q, v in enumerate(ins["imm"]):
                arr[k].imm[q] = v
        self._check(self.L.nau_eval(self.h, arr, len(program), result, self._fid(out)))

    def write_vtk(self, path, binary, fields, frame_index=0, time=0.0, params_text=None,
                  variables=(), constants=(), equations=(), domain_text=None):
        """Result frame of the device state (nau_write_vtk; io/vtk.cpp:219-304 layout).
        fields: names in workspace order (r excluded)."""
        m = FrameMeta()
        m.frame_index, m.time = int(frame_index), float(time)
        m.domain_text = domain_text.encode() if domain_text else None
        m.params_text = params_text.encode() if params_text else None
        keep = []
        for attr, items in (("variables", variables), ("constants", constants),
                            ("equations", equations)):
            cnt, arr = _strs(list(items))
            keep.append(arr)
            setattr(m, "n_" + attr, cnt)
            setattr(m, attr, arr)
        ids = (C.c_int * max(1, len(fields)))(*[self._fid(f) for f in fields])
        cnt, names = _strs([f if isinstance(f, str) else f.name for f in fields])
        m.n_fields, m.field_ids, m.field_names = cnt, ids, names
        self._check(self.L.nau_write_vtk(self.h, str(path).encode(), int(binary), C.byref(m)))

    def set_random_state(self, seed, counters=None):
        """≙ the case's RandomState: seed + per-particle draw counters (original order)."""
        ptr = None
        if counters is not None:
            self._rng_keep = np.ascontiguousarray(counters, dtype=np.uint64)
            ptr = _p(self._rng_keep)
        self._check(self.L.nau_set_random_state(self.h, C.c_ulonglong(seed), ptr))

    def random_counters(self):
        out = np.zeros(self.n, dtype=np.uint64)
        self._check(self.L.nau_get_random_counters(self.h, _p(out)))
        return out

    def io_fence(self):
        self._check(self.L.nau_io_fence(self.h))

    def io_join(self):
        self._check(self.L.nau_io_join(self.h))

    def fill(self, f, value):
        v = np.zeros(9)
        vv = np.atleast_1d(np.asarray(value, dtype=np.float64)).ravel()
        v[: vv.size] = vv
        self._check(self.L.nau_fill(self.h, self._fid(f), _p(v)))

    def device_ptr(self, f):
        p = C.c_void_p()
        self._check(self.L.nau_field_device_ptr(self.h, self._fid(f), C.byref(p)))
        return p.value

    # ---- ParticleSystem ----
    def boundary_shift(self):
        self._check(self.L.nau_boundary_shift(self.h))

    def build_cells(self):
        self._check(self.L.nau_build_cells(self.h))

    @property
    def ncells(self):
        return self.L.nau_ncells(self.h)

    @property
    def rebuild_count(self):
        return self.L.nau_rebuild_count(self.h)

    @property
    def warning_count(self):
        return self.L.nau_warning_count(self.h)

    def active(self):
        out = np.empty(self.n, np.uint8)
        self._check(self.L.nau_get_active(self.h, _p(out)))
        return out

    def active_count(self):
        return self.L.nau_active_count(self.h)

    def cell_tables(self):
        nc = self.ncells
        cell_of = np.empty(self.n, np.int32)
        start = np.empty(nc, np.int32)
        count = np.empty(nc, np.int32)
        srt = np.empty(max(1, self.n), np.int32)
        self._check(self.L.nau_cell_tables(self.h, _p(cell_of), _p(start), _p(count), _p(srt)))
        return cell_of, start, count, srt[: int(count.sum())].copy()

    def neighbor_counts(self, radius):
        out = np.empty(self.n, np.int32)
        self._check(self.L.nau_neighbor_counts(self.h, float(radius), _p(out)))
        return out

    # ---- operators ----
    def _operand(self, o):
        x = Operand()
        if isinstance(o, (Field, str)):
            f = self.fields[o] if isinstance(o, str) else o
            x.field_id, x.rows, x.cols = f.id, f.rows, f.cols
        else:
            v = np.atleast_1d(np.asarray(o, dtype=np.float64)).ravel()
            x.field_id, x.rows, x.cols = -1, v.size, 1
            for k, val in enumerate(v):
                x.value[k] = val
        return x

    def interact(self, name, operands, out, kernel=None):
        """Evaluate SFL operator `name` for all particles into field `out`.

        operands: the kOps[] operand list WITHOUT the kernel keyword (fields by
        name/Field, uniforms as numbers or tuples); kernel: keyword such as
        "Wp53220" or "Wc33220" for SPH operators.
        """
        op = OPS[name]
        kf, kd = (K_WENDLAND, self.dim) if kernel is None else decode_kernel(kernel)
        arr = (Operand * len(operands))(*[self._operand(o) for o in operands])
        self._check(self.L.nau_interact(self.h, op, kf, kd, arr, len(operands), self._fid(out)))

    def interact_g11_l0(self, operands, out_g, out_l, kernel=None):
        """out_g = sph_G11(operands); out_l = sph_L0(operands), in that order — one fused
        list walk in FAST mode (nau_interact_g11_l0), else the two interact() calls."""
        kf, kd = (K_WENDLAND, self.dim) if kernel is None else decode_kernel(kernel)
        arr = (Operand * len(operands))(*[self._operand(o) for o in operands])
        self._check(self.L.nau_interact_g11_l0(self.h, kf, kd, arr, len(operands),
                                               self._fid(out_g), self._fid(out_l)))

    def euler(self, x, xdot, dt, out):
        self._check(self.L.nau_euler(self.h, self._fid(x), self._fid(xdot), float(dt),
                                     self._fid(out)))

    def symplectic_step(self, v, vdot, mask, dt):
        self._check(self.L.nau_symplectic_step(self.h, self._fid(v), self._fid(vdot),
                                               -1 if mask is None else self._fid(mask), float(dt)))

    def wcsph_step(self, p: WcsphParams):
        self._check(self.L.nau_wcsph_step(self.h, C.byref(p)))

    def set_graphs(self, on):
        """CUDA-graph replay of wcsph_step (nau_set_graphs; default on)."""
        self._check(self.L.nau_set_graphs(self.h, 1 if on else 0))

    def wcsph_pass(self, p: WcsphParams, k: int):
        """0 cells + list + density/EOS, 1 momentum, 2 symplectic update (nau_wcsph_pass)."""
        self._check(self.L.nau_wcsph_pass(self.h, C.byref(p), k))

    def dem_step(self, p: DemParams):
        self._check(self.L.nau_dem_step(self.h, C.byref(p)))

    def leapfrog_step(self, p: GravityParams):
        self._check(self.L.nau_leapfrog_step(self.h, C.byref(p)))

    def reduce(self, kind, f):
        kinds = {"fmax": 0, "fmin": 1, "fsum": 2, "fmean": 3}
        out = np.zeros(9)
        self._check(self.L.nau_reduce(self.h, kinds[kind], self._fid(f), _p(out)))
        return out[: (self._comps(f) if kinds[kind] >= 2 else 1)]

    def sync(self):
        self._check(self.L.nau_sync(self.h))

    # ---- instrumentation ----
    def profile(self, on=True):
        self._check(self.L.nau_profile_enable(self.h, 1 if on else 0))

    def profile_ms(self, cls=1):
        cnt = C.c_long(0)
        ms = self.L.nau_profile_ms(self.h, cls, C.byref(cnt))
        return ms, cnt.value

    @property
    def launches(self):
        return self.L.nau_launch_count(self.h)

    def list_stats(self):
        """dict(walkers, entries, warp_cost, lane_efficiency) of the cached neighbour
        lists (nau_list_stats; synchronises)."""
        out = (C.c_double * 3)()
        self._check(self.L.nau_list_stats(self.h, out))
        return {"walkers": out[0], "entries": out[1], "warp_cost": out[2],
                "entries_per_walker": out[1] / max(out[0], 1.0),
                "lane_efficiency": out[1] / max(out[2], 1.0)}

    @property
    def wcsph_path(self):
        """Kernels of the last wcsph_step: dict(fast, source, images) (nau_wcsph_path)."""
        v = self.L.nau_wcsph_path(self.h)
        if v < 0:
            return None
        return {"fast": bool(v & 16), "source": ("sweep", "lists", "paired")[(v >> 2) & 3],
                "images": bool(v & 1)}


class Case:
    """The device equation executor (nau_case_*, csrc/executor.cpp): an arbitrary deck's
    equation list solved with Case::solve_step semantics (case.cpp:9-67) on a Context.
    Symbols: constants/variables are uniform tensors, fields name Context fields."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        self.L = ctx.L
        h = C.c_void_p()
        st = self.L.nau_case_create(ctx.h, C.byref(h))
        if st != 0:
            raise NauError(st, "nau_case_create: set particles first")
        self.h = h
        if not hasattr(ctx, "_cases"):
            ctx._cases = []
        ctx._cases.append(self)
        for name, f in ctx.fields.items():
            if name != "r":
                self._check(self.L.nau_case_field(self.h, name.encode(), f.id))

    def _check(self, st):
        if st != 0:
            bad = C.c_long(-1)
            msg = self.L.nau_case_last_error(self.h, C.byref(bad)).decode()
            raise NauError(st, msg, bad.value)

    @staticmethod
    def _tensor(value):
        a = np.asarray(value, dtype=np.float64)
        if a.ndim == 0:
            a = a.reshape(1, 1)
        elif a.ndim == 1:
            a = a.reshape(-1, 1)  # a python vector is a column
        flat = np.zeros(9)
        flat[: a.size] = a.ravel(order="F")
        return a.shape[0], a.shape[1], flat

    def constant(self, name, value):
        r, c, v = self._tensor(value)
        self._check(self.L.nau_case_constant(self.h, name.encode(), r, c, _p(v)))
        return self

    def variable(self, name, value):
        r, c, v = self._tensor(value)
        self._check(self.L.nau_case_variable(self.h, name.encode(), r, c, _p(v)))
        return self

    def set_variable(self, name, value):
        r, c, v = self._tensor(value)
        self._check(self.L.nau_case_set_variable(self.h, name.encode(), r, c, _p(v)))

    def get_variable(self, name):
        v = np.zeros(9)
        r, c = C.c_int(0), C.c_int(0)
        self._check(self.L.nau_case_get_variable(self.h, name.encode(), _p(v), C.byref(r),
                                                 C.byref(c)))
        return v[: r.value * c.value].reshape(c.value, r.value).T.copy()

    def field(self, name, fid=None):
        f = self.ctx.fields[name] if fid is None else fid
        self._check(self.L.nau_case_field(self.h, name.encode(), self.ctx._fid(f)))
        return self

    def equation(self, name, text):
        self._check(self.L.nau_case_equation(self.h, name.encode(), text.encode()))
        return self

    def solve_equation(self, k):
        self._check(self.L.nau_case_solve_equation(self.h, k))

    def solve_step(self):
        self._check(self.L.nau_case_solve_step(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.L.nau_case_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
