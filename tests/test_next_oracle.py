"""CPU: the oracle's restatement of the SURVEY.md section 8(f) rows pinned
against the reference's own outputs (tests/golden/next.npz, made by
tests/golden/make_golden_next.py): deferred_baseline, FHV1 snapshot bytes,
rebuild_pofl_as_pofa."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2211_15460_b200.lights import Light, headlight
from paper_2211_15460_b200.raster import CaptureStrategy, RasterConfig
from paper_2211_15460_b200.scene import Camera, capture_camera, viewpoint_camera
from tests._golden import BUILTINS, golden_scene, npz, sha

CAMS = {
    "px_persp": lambda: viewpoint_camera("+x", (40, 32), "perspective"),
    "pz_ortho": lambda: viewpoint_camera("+z", (36, 36), "orthographic"),
    "py_persp": lambda: viewpoint_camera("+y", (32, 28), "perspective", fov_deg=50.0, distance=1.2),
    # inside the unit cube: triangles behind the eye are skipped (fhv/raster.py:189-190)
    "near_persp": lambda: Camera("perspective", np.array([0.5, 0.45, 0.62]), np.array([0.1, 0.05, -1.0]),
                                 np.array([0.0, 1.0, 0.0]), 75.0, (48, 40), 0.01, 2.0),
}


def lights_for(lname, cam):
    if lname == "head":
        return [headlight(cam)]
    return [Light("directional", direction=np.array([0.3, 0.8, 0.5]), color=(0.9, 0.8, 0.7),
                  ambient=(0.05, 0.05, 0.05)),
            Light("point", position=np.array([0.5, 1.4, 0.6]), color=(0.6, 0.6, 0.9),
                  ambient=(0.02, 0.03, 0.04))]


def background(lname):
    return (0.1, 0.2, 0.3, 0.5) if lname == "two" else (0.0, 0.0, 0.0, 0.0)


# colours go through pow (libm here and in the reference): stated bound 1e-12 absolute
TOL = 1e-12


@pytest.mark.parametrize("name", BUILTINS)
@pytest.mark.parametrize("cname", sorted(CAMS))
@pytest.mark.parametrize("lname", ("head", "two"))
def test_deferred_oracle_matches_reference(name, cname, lname):
    s = golden_scene(name)
    cam = CAMS[cname]()
    out = orc.deferred(s, cam, lights_for(lname, cam), background(lname))
    g = npz("next")
    k = f"{name}/deferred/{cname}/{lname}/"
    assert np.array_equal(out["depth"], g[k + "depth"])
    for f in ("gpos", "gnrm", "gmat", "gobj", "valid"):
        assert np.array_equal(out[f], g[k + f]), f
    np.testing.assert_allclose(out["rgba"], g[k + "rgba"], rtol=0, atol=TOL)


def test_deferred_near_camera_skips_triangles_behind_eye():
    s = golden_scene("cornell")
    cam = CAMS["near_persp"]()
    out = orc.deferred(s, cam, lights_for("head", cam))
    assert out["valid"].any() and not out["valid"].all()


@pytest.mark.parametrize("name", BUILTINS)
def test_snapshot_bytes_match_reference(name):
    s = golden_scene(name)
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 32))
    g = npz("next")
    vols = {"ppfl": orc.build_ppfl(s, cfg), "pofl": orc.build_pofl(s, CaptureStrategy.normal_space(), cfg, 4),
            "pofa": orc.pofa_build(s, CaptureStrategy.normal_space(), cfg, 4)}
    for vname, vol in vols.items():
        blob = orc.snapshot_bytes(vol)
        assert len(blob) == int(g[f"{name}/snapshot/{vname}/len"])
        assert sha(np.frombuffer(blob, np.uint8)) == str(g[f"{name}/snapshot/{vname}/sha"]), vname


@pytest.mark.parametrize("name", BUILTINS)
@pytest.mark.parametrize("st,L", (("normal_space", 4), ("three_way_geometry", 3)))
def test_rebuild_pofl_as_pofa_matches_reference(name, st, L):
    s = golden_scene(name)
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 32))
    rb = orc.rebuild_pofl_as_pofa(orc.build_pofl(s, CaptureStrategy(st), cfg, L))
    g = npz("next")
    k = f"{name}/rebuild/{st}_L{L}/"
    assert rb["next_free"] == int(g[k + "n"])
    for f in ("offsets", "counts", "pyramid"):
        assert np.array_equal(rb[f], g[k + f]), f
    for f in ("position", "normal", "material_id", "object_id", "prev_index"):
        assert sha(rb["pool"][f]) == str(g[k + f + "_sha"]), f
