"""GPU test of the reference-side binding (integration/gpu_case.{hpp,cpp}: GpuCase, the
C++ a maintainer adds to the reference), compiled against the reference's own headers
and linked to the reference build by oracle/Makefile (oracle/_ref/libgpucase.so).

For each of the reference's shipped decks (fixture state from tests/golden/decks.npz):
two reference Cases are built through the reference's public API (Workspace, fields,
constants, variables, parsed equations); one is stepped by Case::solve_step on the CPU,
the other is mirrored by GpuCase and stepped on the GPU, then downloaded back into its
Field::values. Both must agree bitwise (EXACT mode, decks without libm transcendentals)
or within 1e-10 / 1e-6 (1 / 10 steps) otherwise."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle import ref

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "libgpucase.so")
Z = np.load(os.path.join(HERE, "golden", "decks.npz"))
INDEX = json.loads(str(Z["index"]))
BITWISE = {"dam_break_2d", "hot_start_demo", "sampling_1k"}
TOL = {1: 1e-10, 10: 1e-6}


def binding():
    if not os.path.exists(LIB):
        pytest.fail("oracle/_ref/libgpucase.so not built (make -C oracle, needs /root/reference)")
    L = C.CDLL(LIB)
    L.gpucase_create.restype = C.c_void_p
    L.gpucase_create.argtypes = [C.c_void_p, C.c_int, C.c_int]
    for f in (L.gpucase_solve_step, L.gpucase_download):
        f.argtypes = [C.c_void_p]
    L.gpucase_active.argtypes = [C.c_void_p, C.c_void_p]
    L.gpucase_destroy.argtypes = [C.c_void_p]
    L.gpucase_last_error.restype = C.c_char_p
    return L


def ref_case(deck, meta):
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
    return rc


def rel_err(a, b):
    scale = max(np.abs(b).max(initial=0.0), 1e-300)
    return float(np.abs(a - b).max(initial=0.0) / scale)


@pytest.mark.parametrize("fast", [False, True])
@pytest.mark.parametrize("deck", INDEX["decks"])
def test_gpu_case_binding_vs_case_solve_step(deck, fast):
    L = binding()
    meta = json.loads(str(Z[f"{deck}_meta"]))
    cpu, gpu = ref_case(deck, meta), ref_case(deck, meta)
    g = L.gpucase_create(gpu.case_ptr(), 0, int(fast))
    assert g, L.gpucase_last_error().decode()
    try:
        for s in range(1, max(meta["steps"]) + 1):
            cpu.solve_step(1)
            assert L.gpucase_solve_step(g) == 0, L.gpucase_last_error().decode()
            if s not in meta["steps"]:
                continue
            assert L.gpucase_download(g) == 0, L.gpucase_last_error().decode()
            act = np.zeros(cpu.n, np.uint8)
            assert L.gpucase_active(g, act.ctypes.data_as(C.c_void_p)) == 0
            np.testing.assert_array_equal(act, cpu.active())
            exact = deck in BITWISE and not fast
            for name, _ in meta["fields"]:
                a, b = gpu.get(name), cpu.get(name)
                if exact:
                    np.testing.assert_array_equal(a, b, err_msg=f"step {s} {name}")
                else:
                    assert rel_err(a, b) <= TOL[s], (s, name)
            for name, _ in meta["variables"]:
                a = ref.AssembledCase.get_variable(gpu, name)
                b = ref.AssembledCase.get_variable(cpu, name)
                if exact:
                    np.testing.assert_array_equal(a, b, err_msg=f"step {s} {name}")
                else:
                    assert rel_err(a, b) <= TOL[s], (s, name)
    finally:
        L.gpucase_destroy(g)
