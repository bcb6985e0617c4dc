"""Pin the CPU oracle (oracle/fhv_oracle.c) against golden vectors produced
by the reference itself (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2211_15460_b200 import sample_scenes
from paper_2211_15460_b200.lights import Light, headlight
from paper_2211_15460_b200.raster import CaptureStrategy, RasterConfig
from paper_2211_15460_b200.scene import capture_camera, viewpoint_camera
from tests._golden import BUILTINS, golden_scene, meta, npz, sha

STRATS = ("one_view", "three_separate", "three_way_geometry", "normal_space")


@pytest.mark.parametrize("name", BUILTINS + ("cube972",))
def test_scene_builders_match_reference(name):
    g = npz("scenes")
    s = sample_scenes.cube972() if name == "cube972" else sample_scenes.builtin_scene(name)
    for k in ("positions", "normals", "face_normals", "material_id", "object_id"):
        assert np.array_equal(getattr(s, k), g[f"{name}/{k}"]), k
    for axis in ("+x", "+y", "+z"):
        for res in (32, 64, 256):
            cfg = RasterConfig.from_camera(capture_camera(s, axis, res))
            assert np.array_equal(cfg.projection, g[f"{name}/proj{axis}{res}"])


@pytest.mark.parametrize("name", BUILTINS)
@pytest.mark.parametrize("res", (32, 64))
@pytest.mark.parametrize("strategy", STRATS)
def test_capture_list_bit_exact(name, res, strategy):
    s = golden_scene(name)
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", res))
    out = orc.capture_list(s, CaptureStrategy(strategy), cfg)
    g = npz("captures")
    k = f"{name}/{res}/list/{strategy}"
    st = g[k + "/stats"]
    assert [out["stats"][x] for x in ("fragments_emitted", "triangles_processed", "passes",
                                      "draw_batches")] == list(st)
    if st[0]:
        assert sha(out["raster_x"]) == str(g[k + "/px_sha"])
        assert sha(out["raster_y"]) == str(g[k + "/py_sha"])
        assert sha(out["world_position"]) == str(g[k + "/wpos_sha"])
        assert sha(out["world_normal"]) == str(g[k + "/wnrm_sha"])


def _check_pool(pool, n, g, prefix):
    for k in ("position", "normal", "material_id", "object_id", "prev_index"):
        assert sha(pool[k][:n]) == str(g[prefix + k + "_sha"]), prefix + k


@pytest.mark.parametrize("name", BUILTINS)
@pytest.mark.parametrize("res", (32, 64, 256))
def test_stores_bit_exact(name, res):
    s = golden_scene(name)
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", res))
    g = npz("captures")
    pp = orc.build_ppfl(s, cfg)
    k = f"{name}/{res}/ppfl/"
    assert [pp["next_free"], pp["capacity"], int(pp["overflowed"])] == list(g[k + "meta"])
    _check_pool(pp["pool"], min(pp["next_free"], pp["capacity"]), g, k)
    assert sha(pp["heads"]) == str(g[k + "heads_sha"])
    small = max(1, pp["next_free"] // 3)
    po = orc.build_ppfl(s, cfg, capacity=small)
    k = f"{name}/{res}/ppfl_small/"
    assert [po["next_free"], po["capacity"], int(po["overflowed"])] == list(g[k + "meta"])
    _check_pool(po["pool"], min(po["next_free"], po["capacity"]), g, k)
    assert sha(po["heads"]) == str(g[k + "heads_sha"])
    for st, L in (("normal_space", 4), ("one_view", 4), ("three_way_geometry", 3)):
        pl = orc.build_pofl(s, CaptureStrategy(st), cfg, L)
        k = f"{name}/{res}/pofl_{st}_L{L}/"
        assert [pl["next_free"], pl["capacity"], int(pl["overflowed"])] == list(g[k + "meta"])
        _check_pool(pl["pool"], min(pl["next_free"], pl["capacity"]), g, k)
        assert sha(pl["heads"]) == str(g[k + "heads_sha"])
        assert np.array_equal(pl["pyramid"], g[k + "pyramid"])
        pa = orc.pofa_build(s, CaptureStrategy(st), cfg, L)
        k = f"{name}/{res}/pofa_{st}_L{L}/"
        _check_pool(pa["pool"], pa["next_free"], g, k)
        assert np.array_equal(pa["offsets"], g[k + "offsets"])
        assert np.array_equal(pa["counts"], g[k + "counts"])
        assert np.array_equal(pa["pyramid"], g[k + "pyramid"])
        assert list(pa["stats"].values()) == list(g[k + "stats"])


def test_appendix_b_table():
    """SURVEY Appendix B fragment-count table, reproduced by the oracle."""
    import hashlib
    for row in meta()["appendix_b"]:
        s = golden_scene(row["scene"])
        cfg = RasterConfig.from_camera(capture_camera(s, "+z", row["res"]))
        if row["res"] == 256:
            continue  # covered by test_stores_bit_exact; keep this test fast
        for st in STRATS:
            assert orc.capture_list(s, CaptureStrategy(st), cfg)["stats"]["fragments_emitted"] == row[st]
        v = orc.pofa_build(s, CaptureStrategy.normal_space(), cfg, 6)
        assert int((v["counts"] > 0).sum()) == row["occupied_L6"]
        assert hashlib.sha1(v["counts"].tobytes()).hexdigest()[:12] == row["counts_sha1_L6"]


def test_c1_cube972():
    s = golden_scene("cube972")
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 256))
    g = npz("c1")
    pp = orc.build_ppfl(s, cfg)
    assert pp["next_free"] == meta()["c1_fragments"] == 83232
    _check_pool(pp["pool"], pp["next_free"], g, "ppfl/")
    assert sha(pp["heads"]) == str(g["ppfl/heads_sha"])
    cam = viewpoint_camera("+x", (256, 256), "perspective")
    rgba, depth, _ = orc.splat(pp["pool"], pp["next_free"], cam, [headlight(cam)], 1.0 / 256, s.materials)
    assert sha(depth) == str(g["splat/depth_sha"])
    np.testing.assert_allclose(rgba, g["splat/rgba"], rtol=0, atol=1e-6)


def _lights(lname, cam):
    if lname == "head":
        return [headlight(cam)]
    return [Light("directional", direction=np.array([0.3, 0.8, 0.5]), color=(0.9, 0.8, 0.7),
                  ambient=(0.05, 0.05, 0.05)),
            Light("point", position=np.array([0.5, 1.4, 0.6]), color=(0.6, 0.6, 0.9),
                  ambient=(0.02, 0.03, 0.04))]


CAMS = {
    "px_persp": lambda: viewpoint_camera("+x", (40, 32), "perspective"),
    "pz_ortho": lambda: viewpoint_camera("+z", (36, 36), "orthographic"),
    "py_persp": lambda: viewpoint_camera("+y", (32, 28), "perspective", fov_deg=50.0, distance=1.2),
}

# Shading tolerance: the reference's splat shades with numpy (libm pow); the
# oracle calls the same libm pow, so it is bit-exact here; ray-cast colours
# carry pow too.  Stated bound for floating-point outputs: 1e-12 absolute.
TOL = 1e-12


@pytest.mark.parametrize("name", BUILTINS)
@pytest.mark.parametrize("cname", sorted(CAMS))
@pytest.mark.parametrize("lname", ("head", "two"))
def test_splat_and_raycast_images(name, cname, lname):
    s = golden_scene(name)
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 32))
    pa = orc.pofa_build(s, CaptureStrategy.normal_space(), cfg, 4)
    pl = orc.build_pofl(s, CaptureStrategy.normal_space(), cfg, 4)
    pp = orc.build_ppfl(s, cfg)
    cam = CAMS[cname]()
    lights = _lights(lname, cam)
    bg = (0.1, 0.2, 0.3, 0.5) if lname == "two" else (0.0, 0.0, 0.0, 0.0)
    g = npz("images")
    for vname, vol in (("pofa", pa), ("ppfl", pp)):
        n = min(vol["next_free"], vol["capacity"])
        rgba, depth, win = orc.splat(vol["pool"], n, cam, lights, 1.0 / 32, s.materials, bg)
        k = f"{name}/splat/{vname}/{cname}/{lname}/"
        assert np.array_equal(depth, g[k + "depth"])
        np.testing.assert_allclose(rgba, g[k + "rgba"], rtol=0, atol=TOL)
        obj = np.where(win >= 0, vol["pool"]["object_id"][np.maximum(win, 0)].astype(np.int32), -1)
        assert np.array_equal(obj, g[k + "obj"])
    if cname == "pz_ortho" and lname == "two":
        return
    for mode in ("opaque_nearest", "transparency", "transparency_shadows"):
        for vname, vol in (("pofa", pa), ("pofl", pl)):
            k = f"{name}/ray/{vname}/{cname}/{lname}/{mode}/"
            radius, eps = g[k + "radius"]
            rgba, stats, ids = orc.raycast(vol, cam, lights, radius, mode=mode, shadow_eps=eps,
                                           materials=s.materials, background=bg, collect_ids=True)
            assert list(stats.values()) == list(g[k + "stats"]), k
            assert np.array_equal(ids, g[k + "ids"])
            np.testing.assert_allclose(rgba, g[k + "rgba"], rtol=0, atol=TOL)


def test_threaded_oracle_matches_sequential():
    """The CPU baseline's threaded oracle: same directory / pyramid / splat
    image, same records per leaf (any order)."""
    s = sample_scenes.sphere_field(8, 3, seed=5, r_lo=0.05, r_hi=0.2, c_lo=0.2, c_hi=0.8)
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 256))
    ns = CaptureStrategy.normal_space()
    ref = orc.pofa_build(s, ns, cfg, 6)
    with orc.threads(4):
        mt = orc.pofa_build(s, ns, cfg, 6)
    for k in ("counts", "offsets", "pyramid"):
        assert np.array_equal(mt[k], ref[k]), k
    assert mt["next_free"] == ref["next_free"]
    key = lambda pool, a, b: np.sort(  # noqa: E731
        pool["position"][a:b].view(np.uint32).astype(np.uint64) @ np.array([1 << 40, 1 << 20, 1], np.uint64))
    off, cnt = ref["offsets"].astype(np.int64), ref["counts"].astype(np.int64)
    for c in np.nonzero(cnt)[0]:
        a, b = off[c], off[c] + cnt[c]
        assert np.array_equal(key(mt["pool"], a, b), key(ref["pool"], a, b))
    cam = viewpoint_camera("+x", (96, 80), "perspective")
    lights = [headlight(cam)]
    r1 = orc.splat(ref["pool"], ref["next_free"], cam, lights, 1 / 256, s.materials)
    with orc.threads(3):
        r2 = orc.splat(ref["pool"], ref["next_free"], cam, lights, 1 / 256, s.materials)
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)
