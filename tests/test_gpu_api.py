"""The north-star facade (``api.capture(scene, variant=...)`` /
``api.reconstruct(fhv, view, method=...)``) against the oracle: every variant
captured bit-exactly, both reconstruction methods matching the reference's
image (depth bit-exact, rgba within 1e-12, ray-cast statistics exact)."""
import numpy as np
import pytest

import paper_2211_15460_b200 as fhv
from oracle import oracle as orc
from paper_2211_15460_b200 import api
from paper_2211_15460_b200.lights import headlight
from paper_2211_15460_b200.render import image_numpy
from paper_2211_15460_b200.scene import capture_camera, viewpoint_camera

pytestmark = pytest.mark.gpu

RES = (48, 40)  # RasterConfig resolution: a 40 x 40 capture grid (fhv/raster.py:359)


def _cfg(scene):
    cam = capture_camera(scene, "+z", RES[1])
    return fhv.RasterConfig(RES, fhv.RasterConfig.from_camera(cam).projection, extent=1.0)


@pytest.mark.parametrize("name", ("cornell", "icosphere"))
def test_capture_variants_match_oracle(name):
    s = fhv.sample_scenes.builtin_scene(name)
    cfg = _cfg(s)
    ns = fhv.CaptureStrategy.normal_space()
    pa = api.capture(s, "POFA", resolution=RES, levels=5)
    ra = orc.pofa_build(s, ns, cfg, 5)
    assert pa.layout == "POFA" and pa.pool.next_free == ra["next_free"]
    h = pa.pool.numpy()
    for k in ("position", "normal", "material_id", "object_id", "prev_index"):
        assert np.array_equal(h[k], ra["pool"][k]), k  # the facade's POFA is the reference's exact order
    assert np.array_equal(pa.directory.offsets.cpu().numpy(), ra["offsets"])
    pl = api.capture(s, "pofl", resolution=RES, levels=5, exact_order=True)
    rl = orc.build_pofl(s, ns, cfg, 5)
    assert pl.pool.next_free == rl["next_free"]
    assert np.array_equal(pl.directory.heads.cpu().numpy(), rl["heads"])
    pp = api.capture(s, "PPFL", resolution=RES, exact_order=True)
    rp = orc.build_ppfl(s, cfg)
    assert pp.pool.next_free == rp["next_free"]
    assert np.array_equal(pp.directory.heads.cpu().numpy(), rp["heads"])
    with pytest.raises(ValueError):
        api.capture(s, "voxels", resolution=RES)


@pytest.mark.parametrize("name", ("cornell", "icosphere"))
def test_reconstruct_methods_match_oracle(name):
    s = fhv.sample_scenes.builtin_scene(name)
    cfg = _cfg(s)
    vol = api.capture(s, "POFA", resolution=RES, levels=5)
    ref = orc.pofa_build(s, fhv.CaptureStrategy.normal_space(), cfg, 5)
    view = viewpoint_camera("+x", (56, 44), "perspective")
    lights = [headlight(view)]
    img = image_numpy(api.reconstruct(vol, view, "splat"))
    rgba, depth, _ = orc.splat(ref["pool"], ref["next_free"], view, lights, 1.0 / RES[1], s.materials)
    assert np.array_equal(img.depth, depth)
    assert np.max(np.abs(img.pixels - rgba)) <= 1e-12
    im, st = api.reconstruct(vol, view, "raycast")
    rc = fhv.default_raycast_config(vol)
    orgba, ost, _ = orc.raycast(ref, view, lights, rc.splat_radius_world, materials=s.materials)
    assert st.as_dict() == ost
    assert np.max(np.abs(im.pixels.cpu().numpy() - orgba)) <= 1e-12
    with pytest.raises(ValueError):
        api.reconstruct(vol, view, "voxels")
