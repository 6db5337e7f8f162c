"""CPU tests of the seeded synthetic inputs (paper_1710_08259_b200/scenes.py)."""
import numpy as np

from paper_1710_08259_b200 import scenes


def test_dem_column_rsa_non_overlapping_and_seeded():
    """BASELINE cfg3 inputs at reduced size: random sequential addition gives a
    non-overlapping packing inside the column, untruncated log-normal radii, and the
    same positions for the same seed (different for another seed)."""
    n, s = 20000, (20000 / 2e6) ** (1 / 3)
    box = (0.3 * s, 0.3 * s, 1.2 * s)
    a = scenes.dem_column(n=n, box=box)
    b = scenes.dem_column(n=n, box=box)
    c = scenes.dem_column(n=n, box=box, seed=4)
    np.testing.assert_array_equal(a.pos, b.pos)
    assert not np.array_equal(a.pos, c.pos)
    R, x = a.fields["R"], a.pos
    assert np.all(x - R >= 0) and np.all(x + R <= np.asarray(box)[:, None])
    # brute-force overlap check on a hash of 2 max R
    cs = 2 * R.max()
    key = np.floor(x / cs).astype(np.int64)
    cells = {}
    for i in range(n):
        cells.setdefault(tuple(key[:, i]), []).append(i)
    for cell, idx in cells.items():
        near = []
        for off in np.stack(np.meshgrid([-1, 0, 1], [-1, 0, 1], [-1, 0, 1])).reshape(3, -1).T:
            near += cells.get(tuple(np.asarray(cell) + off), [])
        near = np.asarray(near)
        for i in idx:
            d = np.linalg.norm(x[:, near] - x[:, i:i + 1], axis=0)
            ok = (near == i) | (d >= R[near] + R[i])
            assert ok.all(), (i, near[~ok])
    # the radii are the untruncated log-normal draws (median 1 mm, sigma_log 0.2)
    z = np.log(R / 1e-3) / 0.2
    assert abs(np.median(R) - 1e-3) < 3e-5 and 3.0 < z.max() < 6.0
