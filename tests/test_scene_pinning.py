"""The big bench scenes and their capture setup pinned to the REFERENCE
(tests/golden/scenes_big.json, made by tests/golden/make_golden_scenes.py
from the reference's own ``icosphere`` / ``make_triangle``, ``capture_camera``,
``ortho_projection`` and ``world_pixel_footprint``).

``sample_scenes.sphere_field`` builds the sphere fields struct-of-arrays; here
its arrays must be byte-identical to the reference-built scenes, and
``raster.capture_plan`` (shared by the product and the oracle driver) must
give the reference's pitch and axis projections for the 1920x1080 configs of
C2-C5.  CPU only (the ingest case raises before any device work)."""
import json
import os

import numpy as np
import pytest

import paper_2211_15460_b200 as fhv
from paper_2211_15460_b200 import sample_scenes
from paper_2211_15460_b200.raster import CaptureStrategy, RasterConfig, capture_plan
from paper_2211_15460_b200.scene import capture_camera
from tests._golden import GOLDEN, sha

META = json.load(open(os.path.join(GOLDEN, "scenes_big.json")))
BUILD = {"scatter1m": sample_scenes.scatter1m, "spheres100k": sample_scenes.spheres100k}
_CACHE: dict = {}


def _scene(name):
    if name not in _CACHE:
        _CACHE[name] = BUILD[name]()
    return _CACHE[name]


def _unhex(vals, shape):
    return np.array([float.fromhex(v) for v in vals], dtype=np.float64).reshape(shape)


@pytest.mark.parametrize("name", sorted(BUILD))
def test_big_scene_arrays_match_reference_built(name):
    s = _scene(name)
    g = META["scenes"][name]
    assert s.n_triangles == g["n_triangles"]
    assert sha(s.positions) == g["positions_sha"]
    assert sha(s.normals) == g["normals_sha"]
    assert sha(s.face_normals) == g["face_normals_sha"]
    assert sha(s.material_id) == g["material_id_sha"]
    assert sha(s.object_id) == g["object_id_sha"]
    assert sha(np.array([m.diffuse for m in s.materials], np.float64)) == g["mat_diffuse_sha"]
    assert sha(np.array([m.alpha for m in s.materials], np.float64)) == g["mat_alpha_sha"]


@pytest.mark.parametrize("name", sorted(BUILD))
def test_1080_capture_setup_matches_reference(name):
    s = _scene(name)
    g = META["scenes"][name]
    cam = capture_camera(s, "+z", 1080)
    cfg = RasterConfig((1920, 1080), RasterConfig.from_camera(cam).projection, extent=1.0)
    assert np.array_equal(cfg.projection, _unhex(g["cfg_projection"], (4, 4)))
    ns = capture_plan(s, CaptureStrategy.normal_space(), cfg)
    assert ns.res == g["capture_res"] == 1080
    assert ns.pitch == float.fromhex(g["pitch"])
    for strat in ("three_separate", "three_way_geometry"):
        plan = capture_plan(s, CaptureStrategy(strat), cfg)
        for i, a in enumerate(("+x", "+y", "+z")):
            assert np.array_equal(plan.proj[i], _unhex(g["axis_projection"][a], (4, 4))), (strat, a)
    one = capture_plan(s, CaptureStrategy.one_view(), cfg)
    assert np.array_equal(one.proj[0], _unhex(g["axis_projection"]["+z"], (4, 4)))


def test_zero_length_vertex_normal_raises_like_reference(tmp_path):
    case = META["zero_vn"]
    p = tmp_path / "z.obj"
    p.write_text(case["text"])
    with pytest.raises(fhv.SceneError) as ei:
        fhv.load_scene(str(p))
    assert type(ei.value).__name__ == case["type"] == "SceneError"  # not the later line's SceneLoadError
    assert str(ei.value) == case["message"]
