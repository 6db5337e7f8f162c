"""CPU tests: the C-ABI library loads and exports every symbol include/*.h declares,
and the host-side registry mirrors the reference's kOps[] (no GPU compute here)."""
import os
import re
import subprocess

import pytest

from paper_1710_08259_b200 import nau

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if not h.endswith(".h"):
            continue
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(nau_[a-z0-9_]+)\s*\(", text))
    return names


def exported_symbols():
    out = subprocess.run(["nm", "-D", "--defined-only", nau.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(nau.LIB_PATH):
        pytest.fail("libnau_b200.so not built (run __graft_entry__.build())")
    return nau.load()


def test_every_declared_symbol_is_exported(lib):
    declared = declared_functions()
    assert len(declared) >= 30
    missing = declared - exported_symbols()
    assert not missing, f"declared but not exported: {sorted(missing)}"
    assert declared == set(nau.EXPORTS)


def test_registry_mirrors_reference_kops(lib):
    # /root/reference/proj/src/interactions.cpp:259-269
    expect = {
        "sph_S": (5, 5, 3, 4, True), "sph_D00": (5, 5, 3, 4, True),
        "sph_G11": (5, 5, 3, 4, True), "sph_L0": (5, 5, 3, 4, True),
        "sph_A": (5, 5, 3, 4, True), "dem_l": (7, 7, -1, 6, True),
        "dem_boundary_force": (7, 7, -1, 6, True), "nbody_gravity": (2, 3, -1, -1, False),
        "dem_lsd": (7, 7, -1, 6, True), "sfm": (10, 10, -1, -1, True),
    }
    for name, (amin, amax, ks, rs, fin) in expect.items():
        info = nau.find_interaction(name)
        assert (info["arity_min"], info["arity_max"], info["kernel_slot"], info["radius_slot"],
                info["finite_influence"]) == (amin, amax, ks, rs, fin)
    with pytest.raises(nau.NauError):
        nau.find_interaction("sfm_unknown")


def test_kernel_keywords(lib):
    assert nau.decode_kernel("Wp52220") == (nau.K_WENDLAND, 2)
    assert nau.decode_kernel("Wp53220") == (nau.K_WENDLAND, 3)
    assert nau.decode_kernel("Wc33220") == (nau.K_CUBIC, 3)
    with pytest.raises(nau.NauError) as e:  # test_kernel.cpp:43 lists registered keywords
        nau.decode_kernel("Wx99999")
    assert "Wp52220" in str(e.value)


def test_sm100a_code_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", nau.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
