"""CPU: the oracle's restatement of the reference's operator module and
pyramid helpers reproduces the reference's outputs (tests/golden/scalar.npz,
made by tests/golden/make_golden_scalar.py), and the golden file is
self-consistent for the GPU tests that read it."""
import numpy as np
import pytest

import paper_2211_15460_b200 as fhv
from oracle import oracle
from paper_2211_15460_b200 import raycast
from paper_2211_15460_b200.scene import viewpoint_camera
from tests._golden import npz


@pytest.fixture(scope="module")
def g():
    return npz("scalar")


def test_coverage_oracle_matches_reference(g):
    w, h = (int(v) for v in g["cov/wh"])
    for i, t in enumerate(g["cov/tris"]):
        px, py, lam = oracle.coverage(*[float(v) for v in t], w, h)
        assert np.array_equal(px, g[f"cov/{i}/px"]) and np.array_equal(py, g[f"cov/{i}/py"])
        assert np.array_equal(lam, g[f"cov/{i}/l"].reshape(-1, 3))
    assert int(g["cov/cw_raises"][0]) == 1
    with pytest.raises(ValueError):
        oracle.coverage(0.0, 0.0, 0.0, 10.0, 10.0, 0.0, w, h)


def test_linked_insert_oracle_matches_reference(g):
    heads = np.full(50, -1, np.int32)
    heads[:10] = np.arange(10, dtype=np.int32)
    prev = np.full(400, -7, np.int32)
    oracle.linked_insert(g["li/keys"], heads, prev, 40)
    assert np.array_equal(heads, g["li/heads"]) and np.array_equal(prev, g["li/prev"])


@pytest.mark.parametrize("case", ["ok", "bad"])
def test_pofa_scatter_oracle_matches_reference(g, case):
    cur = np.zeros(40, np.uint32)
    codes = g[f"ps/{case}/codes"]
    dest = np.full(len(codes), -3, np.int64)
    bad = oracle.pofa_scatter(codes, g["ps/offsets"], g["ps/counts"], cur, dest)
    assert bad == int(g[f"ps/{case}/bad"][0])
    assert (bad >= 0) == (case == "bad")
    assert np.array_equal(cur, g[f"ps/{case}/cursors"]) and np.array_equal(dest, g[f"ps/{case}/dest"])


def test_set_paths_and_occupancy_oracle(g):
    L = 4
    levels = [np.zeros(8 ** k, np.uint8) for k in range(L)]
    oracle.set_paths(levels, g["sp/codes"], L)
    assert np.array_equal(np.concatenate(levels), g["sp/pyr"])
    pyr = oracle.pyramid_from_occupancy(g["occ/in"], L)
    assert np.array_equal(pyr, g["occ/pyr"])


def test_scalar_golden_shapes(g):
    n = int(g["ray/n"][0])
    assert n >= 30
    for i in range(n):
        assert g[f"ray/{i}/trav"].shape[1] == 3
        assert g[f"ray/{i}/pofa/gather"].shape[1] == 3
    # the closed-form transparency relation of every recorded pixel: alpha in [0, 1]
    for k in g:
        if k.endswith("/rgba"):
            assert 0.0 <= g[k][3] <= 1.0


def test_gen_primary_ray_matches_reference(g):
    cam = viewpoint_camera("+z", (24, 16), "perspective", 45.0, 1.2)
    k = 0
    for iy in range(0, 16, 3):
        for ix in range(0, 24, 4):
            r = fhv.gen_primary_ray(cam, (ix, iy))
            assert np.array_equal(r.origin, g[f"ray/{k}/o"]) and np.array_equal(r.direction, g[f"ray/{k}/d"])
            k += 1
    with pytest.raises(fhv.SceneError):
        fhv.gen_primary_ray(cam, (24, 0))
    with pytest.raises(fhv.SceneError):
        raycast.Ray(np.zeros(3), np.zeros(3))
