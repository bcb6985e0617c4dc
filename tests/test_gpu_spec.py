"""GPU: speculative capture planning (fhv_capture.cu plan()).  A capture with
the same job count as the previous one launches on the previous item
buffers without a host sync; when the new scene needs MORE work items the
library must notice (FHV_RETRY_ITEMS), restore its outputs and re-plan
exactly.  Each case alternates small / large windows with equal triangle
counts and checks the results against the oracle."""
import numpy as np
import pytest
import torch

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


def _fresh_ctx(fn):
    """Run fn in a new host thread: _lib keeps one scratch context per (device,
    thread), so the speculative item planner starts from nothing."""
    import threading
    out = {}

    def run():
        try:
            out["v"] = fn()
        except BaseException as e:  # noqa: BLE001
            out["e"] = e
    t = threading.Thread(target=run)
    t.start()
    t.join()
    if "e" in out:
        raise out["e"]
    return out["v"]


@pytest.mark.parametrize("exact", [True, False])
def test_item_plan_too_small_is_retried_on_a_fresh_context(exact):
    """32 -> 256 with a context that has only ever planned res 32: the
    speculative plan is short by far; the build must notice and re-plan."""
    s = fhv.sample_scenes.cube972()
    ns = CaptureStrategy.normal_space()

    def run():
        out = []
        for res in (32, 256, 32, 256):
            v = fhv.pofa_build(s, ns, _cfg(s, res), 5, exact_order=exact)
            out.append((v.pool.next_free, v.directory.counts.cpu().numpy(), v.pool.numpy()))
        return out
    got = _fresh_ctx(run)
    for (n, counts, h), res in zip(got, (32, 256, 32, 256)):
        ref = orc.pofa_build(s, ns, _cfg(s, res), 5)
        assert n == ref["next_free"]
        assert np.array_equal(counts, ref["counts"])
        if exact:
            for k in ("position", "normal", "material_id", "object_id", "prev_index"):
                assert np.array_equal(h[k], ref["pool"][k]), (res, k)


def _same(a, b):
    assert a.pool.next_free == b.pool.next_free
    assert np.array_equal(a.directory.counts.cpu().numpy(), b.directory.counts.cpu().numpy())
    assert np.array_equal(a.directory.offsets.cpu().numpy(), b.directory.offsets.cpu().numpy())
    assert np.array_equal(a.pyramid.data.cpu().numpy(), b.pyramid.data.cpu().numpy())
    ha, hb = a.pool.numpy(), b.pool.numpy()
    for k in ("position", "normal", "material_id", "object_id", "prev_index"):
        assert np.array_equal(ha[k], hb[k]), k


def test_async_pofa_build_matches_sync():
    s = fhv.sample_scenes.cube972()
    ns = CaptureStrategy.normal_space()
    cfg = _cfg(s, 128)
    ref = fhv.pofa_build(s, ns, cfg, 5, exact_order=True)
    vols = [fhv.pofa_build(s, ns, cfg, 5, exact_order=True, sync=False) for _ in range(3)]
    assert all(v.pending is not None for v in vols)
    for v in vols:
        v.wait()
        assert v.pending is None
        _same(v, ref)


@pytest.mark.parametrize("delta", [-7, 5])
def test_async_pofa_build_wrong_guess_is_rebuilt(delta):
    s = fhv.sample_scenes.cube972()
    ns = CaptureStrategy.normal_space()
    cfg = _cfg(s, 96)
    ref = fhv.pofa_build(s, ns, cfg, 5, exact_order=True)
    ds = fhv.device.device_scene(s)
    key = next(k for k in ds._pofa_totals if k[1] == 5 and k[0][2] == tuple(cfg.resolution))
    ds._pofa_totals[key] = ref.pool.next_free + delta  # a wrong speculation
    v = fhv.pofa_build(s, ns, cfg, 5, exact_order=True, sync=False)
    torch.cuda.synchronize()
    assert fhv.storage.check_ticket(v) == fhv._lib.FHV_STALE
    v.wait()
    _same(v, ref)


def test_two_streams_get_separate_contexts():
    """A splat on a side stream while the next capture runs on the default
    stream: each stream has its own scratch context (control block, item
    buffers), so both results equal their one-stream counterparts."""
    s = fhv.sample_scenes.cube972()
    ns = CaptureStrategy.normal_space()
    cfg = _cfg(s, 192)
    cam = fhv.viewpoint_camera("+x", (160, 120), "perspective")
    lights = lights_for("head", cam)
    ref_vol = fhv.pofa_build(s, ns, cfg, 5, exact_order=True)
    ref_img = fhv.splat_render(ref_vol.pool, cam, lights, 1.0 / 192, s.materials)
    ref_px = ref_img.pixels.cpu().numpy()
    side = torch.cuda.Stream()
    vols = []
    for _ in range(3):
        v = fhv.pofa_build(s, ns, cfg, 5, exact_order=True, sync=False)
        side.wait_stream(torch.cuda.current_stream())
        v.pool.position.record_stream(side)
        with torch.cuda.stream(side):
            img = fhv.splat_render(v.pool, cam, lights, 1.0 / 192, s.materials)
        vols.append((v, img))
    torch.cuda.synchronize()
    for v, img in vols:
        v.wait()
        _same(v, ref_vol)
        assert np.array_equal(img.pixels.cpu().numpy(), ref_px)
    ctxs = {k for k in fhv._lib._ctxs if k[0] == torch.cuda.current_device()}
    assert len({k[2] for k in ctxs}) >= 2  # distinct streams -> distinct contexts


@pytest.mark.parametrize("delta", [0, 9])
def test_async_build_in_a_cuda_graph(delta):
    """pofa_build(sync=False) + the device-side ticket check captured in a
    CUDA graph: every replay re-runs the whole build and is checked
    (acc = [first bad status, replays checked])."""
    s = fhv.sample_scenes.cube972()
    ns = CaptureStrategy.normal_space()
    cfg = _cfg(s, 160)
    ref = fhv.pofa_build(s, ns, cfg, 5, exact_order=True)
    ds = fhv.device.device_scene(s)
    key = next(k for k in ds._pofa_totals if k[1] == 5 and k[0][2] == tuple(cfg.resolution))
    guess = ref.pool.next_free + delta
    ds._pofa_totals[key] = guess
    gs = torch.cuda.Stream()
    acc = torch.zeros(2, dtype=torch.int64, device="cuda")
    tk = torch.zeros(4, dtype=torch.int64).pin_memory()
    lib = fhv._lib.load()

    def step():
        v = fhv.pofa_build(s, ns, cfg, 5, exact_order=True, sync=False, ticket=tk)
        assert lib.fhv_ticket_accumulate(fhv._lib.ctx(v.pool.device), guess, fhv._lib.ptr(acc),
                                         fhv._lib.stream_ptr(v.pool.device)) == 0
        return v
    with torch.cuda.stream(gs):
        step()
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        v = step()
    acc.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    bad, n = acc.cpu().tolist()
    assert n == 3
    if delta == 0:
        assert bad == 0
        _same(v, ref)
    else:
        assert bad == fhv._lib.FHV_STALE
    ds._pofa_totals[key] = ref.pool.next_free


@pytest.mark.parametrize("exact", (False, True))
def test_job_setup_error_survives_pool_guess(exact):
    """A pipelined ``tris=`` buffer that already holds a pool guess: a scene
    whose face normal is not unit must still raise ValueError (tangent_basis,
    fhv/raster.py:147-163) -- pass 1's job-setup status is not cleared before
    pass 2 (the fused fhv_pofa_build path, synchronous and asynchronous)."""
    good = fhv.sample_scenes.cube972()
    ns = CaptureStrategy.normal_space()
    cfg = _cfg(good, 64)
    ds = fhv.device.DeviceScene(good, torch.device("cuda", 0))
    fhv.pofa_build(good, ns, cfg, 4, exact_order=exact, tris=ds)  # stores the guess on ds
    bad_fn = good.face_normals.copy()
    bad_fn[5] *= 2.0
    ds.fnrm.copy_(torch.from_numpy(bad_fn))
    with pytest.raises(ValueError):
        fhv.pofa_build(good, ns, cfg, 4, exact_order=exact, tris=ds)
    with pytest.raises(ValueError):
        fhv.pofa_build(good, ns, cfg, 4, exact_order=exact, tris=ds, sync=False).wait()


def _same_pofl(a, b):
    assert a.pool.next_free == b.pool.next_free
    assert np.array_equal(a.directory.heads.cpu().numpy(), b.directory.heads.cpu().numpy())
    assert np.array_equal(a.pyramid.data.cpu().numpy(), b.pyramid.data.cpu().numpy())
    n = b.pool.stored_count
    ha, hb = a.pool.numpy(), b.pool.numpy()
    for k in ("position", "normal", "material_id", "object_id", "prev_index"):
        assert np.array_equal(ha[k][:n], hb[k][:n]), k


@pytest.mark.parametrize("exact", (True, False))
def test_async_pofl_build_matches_sync(exact):
    """build_pofl(sync=False): the same chains / pyramid / pool as the
    synchronous build (fhv/storage.py:574-587), no host wait until wait()."""
    s = fhv.sample_scenes.cube972()
    ns = CaptureStrategy.normal_space()
    cfg = _cfg(s, 128)
    ref = fhv.build_pofl(s, ns, cfg, 5, exact_order=exact)
    vols = [fhv.build_pofl(s, ns, cfg, 5, exact_order=exact, sync=False) for _ in range(3)]
    assert all(v.pending is not None for v in vols)
    for v in vols:
        v.wait()
        assert v.pending is None
        if exact:
            _same_pofl(v, ref)
        else:  # ordered allocation without the chain fix-up: same multiset of records per leaf
            assert v.pool.next_free == ref.pool.next_free
            assert np.array_equal(v.pyramid.data.cpu().numpy(), ref.pyramid.data.cpu().numpy())


def test_async_pofl_build_wrong_guess_is_rebuilt():
    s = fhv.sample_scenes.cube972()
    ns = CaptureStrategy.normal_space()
    cfg = _cfg(s, 96)
    ref = fhv.build_pofl(s, ns, cfg, 5, exact_order=True)
    ds = fhv.device.device_scene(s)
    key = next(k for k in ds._pofl_totals if k[1] == 5 and k[0][2] == tuple(cfg.resolution))
    ds._pofl_totals[key] = ref.pool.next_free + 3  # a wrong speculation
    v = fhv.build_pofl(s, ns, cfg, 5, exact_order=True, sync=False)
    torch.cuda.synchronize()
    assert fhv.storage.check_ticket(v) == fhv._lib.FHV_STALE
    v.wait()
    _same_pofl(v, ref)


def test_async_pofl_build_and_raycast_in_a_cuda_graph():
    """The C2 step as the bench times it: build_pofl(sync=False) + the device
    ticket check + render_raycast captured once in a CUDA graph; every replay
    re-runs both and the image / RaycastStats equal the synchronous ones."""
    s = fhv.sample_scenes.cube972()
    ns = CaptureStrategy.normal_space()
    cfg = _cfg(s, 160)
    ref = fhv.build_pofl(s, ns, cfg, 5, exact_order=True)
    cam = fhv.viewpoint_camera("+x", (96, 64), "perspective")
    lights = lights_for("head", cam)
    rc = fhv.default_raycast_config(ref)
    rimg, rst = fhv.render_raycast(ref, cam, lights, rc)
    gs = torch.cuda.Stream()
    acc = torch.zeros(2, dtype=torch.int64, device="cuda")
    tk = torch.zeros(4, dtype=torch.int64).pin_memory()
    lib = fhv._lib.load()
    n = ref.pool.next_free

    from paper_2211_15460_b200.device import DeviceShading
    from paper_2211_15460_b200.lights import ImageBuffer
    sh = DeviceShading(s.materials, lights, torch.device("cuda"))
    w, h = cam.resolution
    buf = ImageBuffer(w, h, torch.zeros((h, w, 4), dtype=torch.float64, device="cuda"),
                      torch.empty((h, w), dtype=torch.float64, device="cuda"))

    def step():  # everything the graph replays is device work (no host-side tensor creation)
        v = fhv.build_pofl(s, ns, cfg, 5, exact_order=True, sync=False, ticket=tk)
        assert lib.fhv_ticket_accumulate(fhv._lib.ctx(v.pool.device), n, fhv._lib.ptr(acc),
                                         fhv._lib.stream_ptr(v.pool.device)) == 0
        buf.pixels.zero_()
        img, st = fhv.render_raycast(v, cam, lights, rc, out=buf, sync=False, shading=sh)
        return v, img, st
    with torch.cuda.stream(gs):
        step()
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        v, img, st = step()
    acc.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    bad, k = acc.cpu().tolist()
    assert (bad, k) == (0, 3)
    assert np.array_equal(img.pixels.cpu().numpy(), rimg.pixels.cpu().numpy())
    assert fhv.RaycastStats(*st.counters.cpu().tolist()).as_dict() == rst.as_dict()


_ASYNC_PATHS = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2211_15460_b200 as fhv
from oracle import oracle as orc
from paper_2211_15460_b200.raster import CaptureStrategy
from tests._golden import golden_scene
bad = []
for name in ("cornell", "icosphere"):
    s = golden_scene(name)
    cfg = fhv.RasterConfig.from_camera(fhv.capture_camera(s, "+z", 256))
    ref = orc.pofa_build(s, CaptureStrategy.normal_space(), cfg, 5)
    for _ in range(3):  # the first build plans exactly; the later ones speculate
        v = fhv.pofa_build(s, CaptureStrategy.normal_space(), cfg, 5, exact_order=True, sync=False)
        v.wait()
        got = v.pool.numpy()
        for k in ("position", "normal", "material_id", "object_id", "prev_index"):
            if not np.array_equal(got[k], ref["pool"][k]):
                bad.append((name, k))
        if not np.array_equal(v.directory.offsets.cpu().numpy(), ref["offsets"]):
            bad.append((name, "offsets"))
print("BAD", bad) if bad else print("OK")
"""


@pytest.mark.parametrize("env", ({"FHV_DIR_STREAM": "0"}, {"FHV_FORK_CLEARS": "0", "FHV_FUSED_EXPAND": "0"},
                                 {"FHV_FORK_CLEARS": "1"}))
def test_async_build_paths_bit_exact(env):
    """The asynchronous POFA build's scheduling variants give the reference's
    pool and offsets bit for bit: the emission-rank scan fused into the
    directory launch or run on its own (FHV_DIR_STREAM=0: no tile-total
    directory), the leaf-counter / cursor clears on the side stream (mode 1:
    both at the job setup; default: cursors at the counting pass) or inline,
    the speculative plan's fused or separate item expansion."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _ASYNC_PATHS.format(root=root)], env=dict(os.environ, **env),
                         capture_output=True, text=True, cwd=root, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == "OK", out.stdout[-2000:]


def test_raycast_writes_every_pixel_of_a_reused_buffer():
    """A full-frame ray cast into a reused image buffer overwrites every pixel
    (the bench's steps reuse one buffer without clearing it): a NaN-filled
    buffer ends up equal to a fresh render."""
    s = fhv.sample_scenes.cube972()
    ns = CaptureStrategy.normal_space()
    cfg = _cfg(s, 128)
    vol = fhv.pofa_build(s, ns, cfg, 5, exact_order=True)
    cam = fhv.viewpoint_camera("+x", (96, 64), "perspective")
    lights = lights_for("head", cam)
    import dataclasses
    for mode in ("transparency", "opaque_nearest"):
        rc = dataclasses.replace(fhv.default_raycast_config(vol), mode=mode)
        ref, _ = fhv.render_raycast(vol, cam, lights, rc)
        buf = fhv.ImageBuffer(96, 64, torch.full((64, 96, 4), float("nan"), dtype=torch.float64, device="cuda"),
                              torch.full((64, 96), float("nan"), dtype=torch.float64, device="cuda"))
        got, _ = fhv.render_raycast(vol, cam, lights, rc, out=buf)
        assert not bool(torch.isnan(got.pixels).any()), mode
        assert torch.equal(got.pixels, ref.pixels), mode
