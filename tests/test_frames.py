"""Result frames: the library's legacy-VTK reader against
frames the reference itself wrote (tests/golden/make_vtk_golden.py), and — on the
GPU — the writer byte for byte against the same files, plus a hot-start round trip."""
import os

import numpy as np
import pytest

from paper_1710_08259_b200 import nau

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _case():
    return np.load(os.path.join(GOLD, "frame_case.npz"))


@pytest.mark.parametrize("fmt", ["ascii", "binary"])
def test_reader_matches_reference_frame(fmt):
    z = _case()
    f = nau.read_vtk(os.path.join(GOLD, f"frame_{fmt}.vtk"))
    assert (f["dim"], f["frame"], f["time"]) == (3, 7, 0.125)
    np.testing.assert_array_equal(f["pos"], z["pos"])
    assert list(f["arrays"]) == [str(k) for k in z["field_order"]]
    for k in z["field_order"]:
        shape, soa = f["arrays"][str(k)]
        assert shape == tuple(z["shape_" + str(k)])
        np.testing.assert_array_equal(soa, z["f_" + str(k)])
    np.testing.assert_array_equal(f["rand_counters"], z["active"].astype(np.uint64))
    s = f["strings"]
    assert s["params"] == ["simulated_time=2.5"]
    assert s["field_shapes"] == ["v=3x1", "w2=2x1", "S=3x3"]
    assert s["constants"] == ["g=0|0|-9.81", "k=0.1"]
    assert s["equations"] == ["rhoeq: rho=rho+k*rand(0,1)"]


def test_reader_rejects_non_vtk(tmp_path):
    p = tmp_path / "x.vtk"
    p.write_text("hello\n")
    with pytest.raises(nau.NauError) as e:
        nau.read_vtk(p)
    assert "not a legacy VTK file" in str(e.value)


def _gpu_state(z):
    c = nau.Context(0)
    c.set_domain(3, [0, 0, 0], [2, 2, 2], [0.5, 0.5, 0.5], list(z["kinds"]))
    c.set_particles(z["pos"])
    for k in z["field_order"]:
        k = str(k)
        r, cc = z["shape_" + k]
        c.add_field(k, int(r), int(cc), z["f_" + k])
    c.boundary_shift()
    c.build_cells()  # cell order != original order: the writer must unsort
    c.set_random_state(int(z["seed"]), z["active"].astype(np.uint64))
    return c


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["ascii", "binary"])
def test_writer_byte_identical_to_reference(tmp_path, fmt):
    z = _case()
    gold = os.path.join(GOLD, f"frame_{fmt}.vtk")
    s = nau.read_vtk(gold)["strings"]
    c = _gpu_state(z)
    try:
        np.testing.assert_array_equal(c.active(), z["active"])
        out = tmp_path / "f.vtk"
        c.write_vtk(out, fmt == "binary", [str(k) for k in z["field_order"]], frame_index=7,
                    time=0.125, params_text=s["params"][0], variables=s["variables"],
                    constants=s["constants"], equations=s["equations"])
        assert out.read_bytes() == open(gold, "rb").read()
    finally:
        c.close()


@pytest.mark.gpu
def test_hot_start_round_trip(tmp_path):
    """frame -> read -> fresh context (set_particles / add_field / rand counters) ->
    frame: byte identical (hot start restores the whole per-particle state)."""
    z = _case()
    gold = os.path.join(GOLD, "frame_binary.vtk")
    f = nau.read_vtk(gold)
    c = nau.Context(0)
    try:
        c.set_domain(3, [0, 0, 0], [2, 2, 2], [0.5, 0.5, 0.5], list(z["kinds"]))
        c.set_particles(f["pos"])
        for name, ((r, cc), soa) in f["arrays"].items():
            c.add_field(name, r, cc, soa)
        c.boundary_shift()
        c.set_random_state(int(z["seed"]), f["rand_counters"])
        s = f["strings"]
        out = tmp_path / "g.vtk"
        c.write_vtk(out, True, list(f["arrays"]), frame_index=f["frame"], time=f["time"],
                    params_text=s["params"][0], variables=s["variables"],
                    constants=s["constants"], equations=s["equations"])
        assert out.read_bytes() == open(gold, "rb").read()
    finally:
        c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("fast", [False, True])
def test_split_run_equals_straight_run(tmp_path, fast):
    """3D dam break: 6 steps straight = 3 steps, a BINARY frame, a hot start in a
    fresh context from that frame, 3 more steps — bitwise (the frame restores the
    whole state in original order, so the cell lists and sums are the same)."""
    import test_gpu_parity as tg
    from paper_1710_08259_b200 import scenes
    sc = scenes.dam_break(3, dx=0.02)
    names = ["rho", "p", "v", "vdot", "mask"]
    a = nau.Context(0)
    b = nau.Context(0)
    try:
        pa = tg._gpu_dam(a, sc)
        a.set_mode(fast)
        for _ in range(6):
            a.wcsph_step(pa)
        straight = {k: a.download(k) for k in ["r"] + names}
        pb = tg._gpu_dam(b, sc)
        b.set_mode(fast)
        for _ in range(3):
            b.wcsph_step(pb)
        path = tmp_path / "split.vtk"
        b.write_vtk(path, True, names, frame_index=3, time=3 * sc.params["dt"])
        b.close()
        f = nau.read_vtk(path)
        b = nau.Context(0)
        b.set_domain(sc.dim, sc.min_cells, sc.max_cells, sc.cell_size, sc.kinds)
        b.set_particles(f["pos"])
        for k in names:
            (r, cc), soa = f["arrays"][k]
            b.add_field(k, r, cc, soa)
        b.boundary_shift()
        f_ids = b.fields
        pb.f_rho, pb.f_p, pb.f_v, pb.f_vdot, pb.f_mask = (f_ids["rho"].id, f_ids["p"].id,
                                                          f_ids["v"].id, f_ids["vdot"].id,
                                                          f_ids["mask"].id)
        b.set_mode(fast)
        for _ in range(3):
            b.wcsph_step(pb)
        for k in ["r"] + names:
            np.testing.assert_array_equal(b.download(k), straight[k], err_msg=k)
    finally:
        a.close()
        b.close()
