"""GPU: speculative capture planning (fhv_capture.cu plan()).  A capture with
the same job count as the previous one launches on the previous item
buffers without a host sync; when the new scene needs MORE work items the
library must notice (FHV_RETRY_ITEMS), restore its outputs and re-plan
exactly.  Each case alternates small / large windows with equal triangle
counts and checks the results against the oracle."""
import numpy as np
import pytest

import paper_2211_15460_b200 as fhv
from oracle import oracle as orc
from paper_2211_15460_b200.raster import CaptureStrategy, RasterConfig
from paper_2211_15460_b200.scene import capture_camera
from tests.test_next_oracle import lights_for

pytestmark = pytest.mark.gpu


def _cfg(s, res):
    return RasterConfig.from_camera(capture_camera(s, "+z", res))


@pytest.mark.parametrize("order", ((32, 256, 64, 256), (256, 32, 256)))
def test_pofa_build_retries_when_items_grow(order):
    s = fhv.sample_scenes.cube972()
    ns = CaptureStrategy.normal_space()
    for res in order:
        cfg = _cfg(s, res)
        gpu = fhv.pofa_build(s, ns, cfg, 5, exact_order=True)
        ref = orc.pofa_build(s, ns, cfg, 5)
        assert gpu.pool.next_free == ref["next_free"]
        assert np.array_equal(gpu.directory.counts.cpu().numpy(), ref["counts"])
        h = gpu.pool.numpy()
        for k in ("position", "normal", "material_id", "object_id", "prev_index"):
            assert np.array_equal(h[k], ref["pool"][k]), (res, k)


def test_linked_builds_retry_when_items_grow():
    s = fhv.sample_scenes.cube972()
    for res in (32, 256, 48, 256):
        cfg = _cfg(s, res)
        pp = fhv.build_ppfl(s, cfg, exact_order=True)
        rp = orc.build_ppfl(s, cfg)
        assert pp.pool.next_free == rp["next_free"]
        assert np.array_equal(pp.directory.heads.cpu().numpy(), rp["heads"])
        assert np.array_equal(pp.pool.prev_index[:pp.pool.stored_count].cpu().numpy(),
                              rp["pool"]["prev_index"][:rp["next_free"]])
        pl = fhv.build_pofl(s, CaptureStrategy.normal_space(), cfg, 5, exact_order=True)
        rl = orc.build_pofl(s, CaptureStrategy.normal_space(), cfg, 5)
        assert pl.pool.next_free == rl["next_free"]
        assert np.array_equal(pl.directory.heads.cpu().numpy(), rl["heads"])


def test_deferred_retries_when_items_grow():
    s = fhv.sample_scenes.cube972()
    for res in ((32, 24), (256, 200), (40, 40), (256, 200)):
        cam = fhv.viewpoint_camera("+x", res, "perspective")
        img, gb = fhv.deferred_baseline(s, cam, lights_for("head", cam))
        ref = orc.deferred(s, cam, lights_for("head", cam))
        assert np.array_equal(img.depth.cpu().numpy(), ref["depth"])
        assert np.array_equal(gb.position.cpu().numpy(), ref["gpos"])


def test_pofa_pool_guess_too_small_is_refilled():
    """The Python pool-size guess (last total for this scene/plan) misses when
    the same scene is captured at a higher resolution through a new config."""
    s = fhv.sample_scenes.cube972()
    ns = CaptureStrategy.normal_space()
    a = fhv.pofa_build(s, ns, _cfg(s, 64), 5)
    b = fhv.pofa_build(s, ns, _cfg(s, 256), 5)
    ref = orc.pofa_build(s, ns, _cfg(s, 256), 5)
    assert a.pool.next_free < b.pool.next_free == ref["next_free"]
    assert np.array_equal(b.directory.offsets.cpu().numpy(), ref["offsets"])
