"""Multi-GPU partition on one B200: N shards as threads (ThreadComm loopback)
run the same kernels and exchange code paths as N ranks over NCCL; their
union must be bit-identical to the 1-GPU pofa_build / splat_render."""
import threading

import numpy as np
import pytest
import torch

import paper_2211_15460_b200 as fhv
from paper_2211_15460_b200 import sample_scenes, shard
from paper_2211_15460_b200.render import image_numpy
from paper_2211_15460_b200.scene import look_at_camera

pytestmark = pytest.mark.gpu


def _run_ranks(world, fn):
    comms = shard.ThreadComm.group(world, torch.device("cuda", 0))
    out, err = [None] * world, []

    def go(c):
        try:
            torch.cuda.set_device(0)
            out[c.rank] = fn(c)
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            c.hub.barrier.abort()

    th = [threading.Thread(target=go, args=(c,)) for c in comms]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out


def _scene(name):
    if name == "spheres":
        return sample_scenes.sphere_field(6, 3, seed=3, r_lo=0.05, r_hi=0.2, c_lo=0.2, c_hi=0.8)
    return sample_scenes.builtin_scene(name)


@pytest.mark.parametrize("name", ("cornell", "icosphere", "spheres"))
@pytest.mark.parametrize("world,balance", ((2, False), (3, True), (4, True), (8, False)))
def test_sharded_pofa_and_splat_equal_single_gpu(name, world, balance):
    scene = _scene(name)
    res, L = 256, 6
    cfg = fhv.RasterConfig.from_camera(fhv.capture_camera(scene, "+z", res))
    ns = fhv.CaptureStrategy.normal_space()
    ref = fhv.pofa_build(scene, ns, cfg, L, exact_order=True)
    cam = fhv.viewpoint_camera("+x", (96, 80), "perspective")
    lights = [fhv.headlight(cam)]
    r = 1.0 / res
    ref_img = image_numpy(fhv.splat_render(ref.pool, cam, lights, r, scene.materials))

    def rank_fn(c):
        v = shard.pofa_build_shard(scene, ns, cfg, L, c, balance=balance, exact_order=True)
        img = image_numpy(shard.splat_render_shard(v, cam, lights, r, scene.materials, c))
        pyr = v.gather_pyramid(c)
        return v, img, pyr

    out = _run_ranks(world, rank_fn)
    vols = [o[0] for o in out]
    assert sum(v.pool.capacity for v in vols) == ref.pool.capacity
    assert all(v.total == ref.pool.capacity for v in vols)
    lo = 0
    for v in vols:  # contiguous, complete, in rank order
        assert v.cell_lo == lo
        lo = v.cell_hi
    assert lo == 8 ** L
    cat = lambda f: torch.cat([f(v) for v in vols]).cpu()  # noqa: E731
    assert torch.equal(cat(lambda v: v.directory.counts), ref.directory.counts.cpu())
    assert torch.equal(cat(lambda v: v.directory.offsets), ref.directory.offsets.cpu())
    for k in ("position", "normal", "material_id", "object_id", "prev_index"):
        assert torch.equal(cat(lambda v: getattr(v.pool, k)), getattr(ref.pool, k).cpu()), k
    for v in vols:
        assert v.base == int(ref.directory.offsets[v.cell_lo]) or int(ref.directory.counts[v.cell_lo:v.cell_hi].sum()) == 0
    for _, img, pyr in out:
        assert pyr.equals(ref.pyramid)
        assert np.array_equal(img.depth, ref_img.depth)
        assert np.array_equal(img.pixels, ref_img.pixels)


def test_sharded_fast_order_is_a_per_leaf_permutation():
    scene = _scene("spheres")
    cfg = fhv.RasterConfig.from_camera(fhv.capture_camera(scene, "+z", 256))
    ns = fhv.CaptureStrategy.normal_space()
    ref = fhv.pofa_build(scene, ns, cfg, 6, exact_order=True)
    vols = _run_ranks(2, lambda c: shard.pofa_build_shard(scene, ns, cfg, 6, c))
    # multiset per leaf: sort records inside each leaf range, then compare
    pos = torch.cat([v.pool.position for v in vols]).cpu().numpy()
    rpos = ref.pool.position.cpu().numpy()
    off = ref.directory.offsets.cpu().numpy().astype(np.int64)
    cnt = ref.directory.counts.cpu().numpy().astype(np.int64)
    for c in np.nonzero(cnt)[0][:2000]:
        a = pos[off[c]:off[c] + cnt[c]]
        b = rpos[off[c]:off[c] + cnt[c]]
        assert np.array_equal(a[np.lexsort(a.T)], b[np.lexsort(b.T)])


@pytest.mark.parametrize("name", ("cornell", "spheres"))
@pytest.mark.parametrize("world", (2, 3, 4, 8))
def test_peer_composited_splat_equals_single_gpu(name, world):
    """composite="peer": depth keys / winners RED.MIN'd straight into the
    owning rank's row slab and shaded pixels stored into every rank's frame
    (fhv_splat_peer) -- every rank's frame bit-identical to splat_render of
    the whole pool, twice in a row (buffers reused)."""
    scene = _scene(name)
    res, L = 256, 6
    cfg = fhv.RasterConfig.from_camera(fhv.capture_camera(scene, "+z", res))
    ns = fhv.CaptureStrategy.normal_space()
    ref = fhv.pofa_build(scene, ns, cfg, L, exact_order=True)
    cams = [fhv.viewpoint_camera("+x", (96, 80), "perspective"),
            fhv.viewpoint_camera("+y", (64, 70), "perspective", fov_deg=50.0, distance=1.2)]
    r = 1.0 / res
    bg = (0.1, 0.2, 0.3, 0.5)
    refs = [image_numpy(fhv.splat_render(ref.pool, cam, [fhv.headlight(cam)], r, scene.materials, bg))
            for cam in cams]

    def rank_fn(c):
        v = shard.pofa_build_shard(scene, ns, cfg, L, c, exact_order=True)
        imgs = []
        for cam in cams:
            peer = shard.PeerFrame(*cam.resolution, c, torch.device("cuda", 0))
            for _ in range(2):
                imgs.append(image_numpy(shard.splat_render_shard(v, cam, [fhv.headlight(cam)], r, scene.materials, c,
                                                                 bg, composite="peer", peer=peer)))
        return imgs

    for imgs in _run_ranks(world, rank_fn):
        for i, img in enumerate(imgs):
            want = refs[i // 2]
            assert np.array_equal(img.depth, want.depth)
            assert np.array_equal(img.pixels, want.pixels)


@pytest.mark.parametrize("name", ("cornell", "spheres"))
@pytest.mark.parametrize("world", (2, 4, 8))
@pytest.mark.parametrize("mode", ("opaque_nearest", "transparency"))
def test_subtree_sharded_raycast_equals_single_gpu(name, world, mode):
    """SURVEY 8(e) ray-cast partition: every rank traces only its own octant
    subtrees; opaque = front-most region's first hit (bit-identical),
    transparency = per-region (C, A) partials composited in entry order
    (equal up to reassociation, 1e-12)."""
    scene = _scene(name)
    res, L = 256, 6
    cfg = fhv.RasterConfig.from_camera(fhv.capture_camera(scene, "+z", res))
    ns = fhv.CaptureStrategy.normal_space()
    ref = fhv.pofa_build(scene, ns, cfg, L, exact_order=True)
    cams = [fhv.viewpoint_camera("+x", (96, 80), "perspective"),
            look_at_camera((1.3, 1.1, 1.6), resolution=(72, 64))]
    rc = fhv.default_raycast_config(ref, mode=mode)
    bg = (0.1, 0.2, 0.3, 0.5)
    refs = []
    for cam in cams:
        img, st = fhv.render_raycast(ref, cam, [fhv.headlight(cam)], rc, scene.materials, bg)
        refs.append((img.pixels.cpu().numpy(), st))

    def rank_fn(c):
        v = shard.pofa_build_shard(scene, ns, cfg, L, c, balance=False, exact_order=True)
        outs = []
        for cam in cams:
            img, st = shard.render_raycast_shard(v, cam, [fhv.headlight(cam)], rc, c, scene.materials, bg)
            outs.append((img.pixels.cpu().numpy(), st))
        return outs

    per_rank = _run_ranks(world, rank_fn)
    for i, (want, st_ref) in enumerate(refs):
        hits = sum(o[i][1].hits for o in per_rank)
        assert hits >= st_ref.hits > 0
        for o in per_rank:
            got = o[i][0]
            if mode == "opaque_nearest":
                assert np.array_equal(got, want)
            else:
                assert np.max(np.abs(got - want)) <= 1e-12


@pytest.mark.parametrize("world", (2, 3))
def test_speculative_sharded_build_no_sync(world):
    """pofa_build_shard(sync=False): no host wait and no collective inside the
    build (every rank's total, base and the triangle binning from the first
    synchronous build); wait(comm) checks all tickets -- the union equals the
    1-GPU pofa_build bit for bit, and a rank whose guess is wrong makes EVERY
    rank rebuild (the bases above it were wrong too)."""
    scene = _scene("spheres")
    res, L = 256, 6
    cfg = fhv.RasterConfig.from_camera(fhv.capture_camera(scene, "+z", res))
    ns = fhv.CaptureStrategy.normal_space()
    ref = fhv.pofa_build(scene, ns, cfg, L, exact_order=True)

    def rank_fn(c):
        shard.pofa_build_shard(scene, ns, cfg, L, c, balance=True, exact_order=True)  # fills the guesses
        vols = [shard.pofa_build_shard(scene, ns, cfg, L, c, balance=True, exact_order=True, sync=False)
                for _ in range(2)]
        assert all(v.pending is not None for v in vols)
        for v in vols:
            v.wait(c)
        # a wrong guess on rank 0 shifts every higher rank's base
        ds = fhv.device.device_scene(scene)
        key = next(k for k in ds._shard_totals if k[6] == c.rank and k[7] == c.world)
        good = list(ds._shard_totals[key])
        ds._shard_totals[key] = [good[0] + 5] + good[1:]  # every rank holds the same (wrong) vector
        bad = shard.pofa_build_shard(scene, ns, cfg, L, c, balance=True, exact_order=True, sync=False)
        bad.wait(c)
        return vols[-1], bad

    out = _run_ranks(world, rank_fn)
    for idx in (0, 1):
        vols = [o[idx] for o in out]
        assert sum(v.pool.capacity for v in vols) == ref.pool.capacity
        cat = lambda f: torch.cat([f(v) for v in vols]).cpu()  # noqa: E731
        assert torch.equal(cat(lambda v: v.directory.counts), ref.directory.counts.cpu())
        assert torch.equal(cat(lambda v: v.directory.offsets), ref.directory.offsets.cpu())
        for k in ("position", "normal", "material_id", "object_id", "prev_index"):
            assert torch.equal(cat(lambda v: getattr(v.pool, k)), getattr(ref.pool, k).cpu()), (idx, k)
