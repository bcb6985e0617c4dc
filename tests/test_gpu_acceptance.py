"""GPU: the reference specification's acceptance criteria
and traversal / transmittance examples, run against the
device implementation.  (Criterion 1, the Morton roundtrip, and 9, the
memory formulas, are CPU tests in tests/test_boundary.py.)"""
import numpy as np
import pytest
import torch

import paper_2211_15460_b200 as fhv
from paper_2211_15460_b200 import storage
from paper_2211_15460_b200.lights import Light, headlight
from paper_2211_15460_b200.raster import CaptureStrategy as CS
from paper_2211_15460_b200.raster import RasterConfig
from paper_2211_15460_b200.scene import Material, Scene, capture_camera, make_quad, viewpoint_camera
from tests._golden import BUILTINS, golden_scene

pytestmark = pytest.mark.gpu


def _cfg(s, res):
    return RasterConfig.from_camera(capture_camera(s, "+z", res))


def test_2_ppfl_chains_equal_brute_force_per_pixel_collection():
    s = golden_scene("three-quads")
    cfg = _cfg(s, 32)
    pp = fhv.build_ppfl(s, cfg, exact_order=True)
    lst = fhv.capture_fragments(s, CS.one_view(), cfg)
    px, py = lst["raster_x"].cpu().numpy(), lst["raster_y"].cpu().numpy()
    per_pixel: dict = {}
    for rank, key in enumerate((py.astype(np.int64) * 32 + px).tolist()):
        per_pixel.setdefault(key, []).append(rank)
    heads = pp.directory.heads.cpu().numpy()
    assert set(np.flatnonzero(heads >= 0).tolist()) == set(per_pixel)
    for key, ranks in per_pixel.items():
        # ordered allocation: pool index = emission rank; chains run newest first
        assert fhv.chain_indices(pp.directory.heads, pp.pool.prev_index, key).tolist() == ranks[::-1]


@pytest.mark.parametrize("name", BUILTINS)
def test_3_pofa_structure(name):
    s = golden_scene(name)
    pa = fhv.pofa_build(s, CS.normal_space(), _cfg(s, 64), 6)
    counts = pa.directory.counts.view(torch.int32).cpu().numpy().astype(np.int64)
    offsets = pa.directory.offsets.view(torch.int32).cpu().numpy().astype(np.int64)
    assert np.array_equal(offsets, np.concatenate(([0], np.cumsum(counts)[:-1])))
    assert counts.sum() == pa.pool.next_free == pa.pool.capacity
    codes = np.atleast_1d(storage.cell_code(pa.pool.position.cpu().numpy().astype(np.float64), 6))
    idx = np.arange(len(codes))
    assert np.all((offsets[codes] <= idx) & (idx < offsets[codes] + counts[codes]))  # each slot in its own leaf
    assert np.array_equal(np.bincount(codes, minlength=8 ** 6), counts)               # every slot written once


@pytest.mark.parametrize("name", BUILTINS)
def test_4_cross_layout_equivalence(name):
    s = golden_scene(name)
    cfg = _cfg(s, 64)
    pl = fhv.build_pofl(s, CS.normal_space(), cfg, 5, exact_order=True)
    pa = fhv.pofa_build(s, CS.normal_space(), cfg, 5, exact_order=True)
    heads = pl.directory.heads.cpu().numpy()
    lpos = pl.pool.position.cpu().numpy()
    apos = pa.pool.position.cpu().numpy()
    for code in np.flatnonzero(heads >= 0)[:400]:
        a = apos[pa.leaf_indices(int(code))]
        b = lpos[pl.leaf_indices(int(code))]
        assert sorted(map(tuple, a.tolist())) == sorted(map(tuple, b.tolist()))
    cam = viewpoint_camera("+z", (96, 64), "perspective")
    for mode in fhv.raycast.RAYCAST_MODES:
        ia, sa = fhv.render_raycast(pa, cam, [headlight(cam)], fhv.default_raycast_config(pa, mode=mode))
        il, sl = fhv.render_raycast(pl, cam, [headlight(cam)], fhv.default_raycast_config(pl, mode=mode))
        assert torch.equal(ia.pixels, il.pixels) and sa.as_dict() == sl.as_dict()


def test_5_fig2_composite_closed_form():
    s = golden_scene("three-quads")
    pa = fhv.pofa_build(s, CS.normal_space(), _cfg(s, 64), 4)
    light = Light("directional", direction=np.array([0.0, 0.0, 1.0]))
    ray = fhv.Ray(np.array([0.45, 0.55, 1.5]), np.array([0.0, 0.0, -1.0]))
    rgba = fhv.raycast_pixel(pa, ray, [light], fhv.default_raycast_config(pa))
    # SPEC.md:353,450,563 with the quads' shaded colours R, G, B (front to back red, green, blue)
    assert abs(rgba[3] - 19.0 / 27.0) <= 1e-5
    hits = []
    fhv.raycast_pixel(pa, ray, [light], fhv.default_raycast_config(pa), hit_out=hits)
    assert len(hits) == 3 and [h.t for h in hits] == sorted(h.t for h in hits)
    mats = [s.materials[int(pa.pool.material_id[h.fragment_index])] for h in hits]
    cols = [fhv.shade(pa.pool.position[h.fragment_index].cpu().numpy(), pa.pool.normal[h.fragment_index].cpu().numpy(),
                      m, light, ray.origin) for h, m in zip(hits, mats)]
    expect = cols[0] / 3 + 2 * cols[1] / 9 + 4 * cols[2] / 27
    assert np.allclose(rgba[:3], expect, atol=1e-5)


def test_6_deferred_oracle_object_ids():
    s = golden_scene("icosphere")
    cam = viewpoint_camera("+z", (128, 128), "orthographic")
    lights = [headlight(cam)]
    _, gb = fhv.deferred_baseline(s, cam, lights)
    dref = gb.object_id.cpu().numpy()
    pa = fhv.pofa_build(s, CS.normal_space(), _cfg(s, 128), 6)
    _, _, ids = fhv.render_raycast(pa, cam, lights, fhv.default_raycast_config(pa, mode="opaque_nearest"),
                                   collect_ids=True)
    ids = ids.cpu().numpy()
    both = (dref >= 0) & (ids >= 0)
    assert both.sum() > 1000 and (dref[both] == ids[both]).mean() >= 0.95
    gbs = fhv.render.device_gbuffer(128, 128, pa.pool.device)
    fhv.splat_render(pa.pool, cam, lights, 1.0 / 128, s.materials, id_buffer=gbs)
    sid = gbs.object_id.cpu().numpy()
    both = (dref >= 0) & (sid >= 0)
    assert both.sum() > 1000 and (dref[both] == sid[both]).mean() >= 0.95


@pytest.mark.parametrize("name", ["icosphere", "cornell"])
def test_7_strategy_relations(name):
    s = golden_scene(name)
    res = 64
    cfg = _cfg(s, res)
    n = {k: fhv.capture_fragments(s, CS(k), cfg)["stats"].fragments_emitted for k in fhv.raster.CAPTURE_STRATEGIES}
    assert n["three_separate"] == n["three_way_geometry"]
    P = s.positions
    per = (np.linalg.norm(P[:, 1] - P[:, 0], axis=1) + np.linalg.norm(P[:, 2] - P[:, 1], axis=1)
           + np.linalg.norm(P[:, 0] - P[:, 2], axis=1))
    slack = float(np.sum(2 * per * res))  # footprint = 1 / res
    assert n["one_view"] <= n["normal_space"] + slack
    assert n["normal_space"] <= n["three_way_geometry"] + slack


def test_8_directional_bias():
    s = golden_scene("edge-plane")
    R = 64
    cfg = _cfg(s, R)
    ov = fhv.capture_fragments(s, CS.one_view(), cfg)["stats"].fragments_emitted
    ns = fhv.capture_fragments(s, CS.normal_space(), cfg)["stats"].fragments_emitted
    P = s.positions
    area = 0.5 * np.linalg.norm(np.cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]), axis=1).sum()
    assert ov <= 2 * R
    assert ns >= 0.9 * area * R * R
    lv_ov = fhv.build_pofl(s, CS.one_view(), cfg, 5).pyramid.occupied_leaves().numel()
    lv_ns = fhv.build_pofl(s, CS.normal_space(), cfg, 5).pyramid.occupied_leaves().numel()
    assert lv_ns >= 10 * max(lv_ov, 1)


def test_10_early_termination_soundness_and_effect():
    s = golden_scene("cornell")
    pa = fhv.pofa_build(s, CS.three_way_geometry(), _cfg(s, 64), 5)
    cam = viewpoint_camera("+z", (64, 48), "perspective")
    L = [headlight(cam)]
    i_none, s_none = fhv.render_raycast(pa, cam, L, fhv.default_raycast_config(pa, alpha_cutoff=None))
    i_one, s_one = fhv.render_raycast(pa, cam, L, fhv.default_raycast_config(pa, alpha_cutoff=1.0))
    i_99, s_99 = fhv.render_raycast(pa, cam, L, fhv.default_raycast_config(pa, alpha_cutoff=0.99))
    assert s_99.visited_leaves < s_none.visited_leaves
    assert float((i_one.pixels - i_none.pixels).abs().max()) <= 1e-6


def _slab_scene(alpha):
    m = Material(diffuse=(0.5, 0.5, 0.5), alpha=alpha)
    q = make_quad((0.2, 0.2, 0.5), (0.8, 0.2, 0.5), (0.8, 0.8, 0.5), (0.2, 0.8, 0.5), material_id=0, object_id=1)
    return Scene.from_triangles(q, [m])


@pytest.mark.parametrize("alpha,light_dir,expect", [(1.0, (0.0, 0.0, -1.0), 1.0), (1.0, (0.0, 0.0, 1.0), 0.0),
                                                    (1.0 / 3.0, (0.0, 0.0, 1.0), 2.0 / 3.0)])
def test_11_shadow_transmittance_closed_forms(alpha, light_dir, expect):
    s = _slab_scene(alpha)
    pa = fhv.pofa_build(s, CS.normal_space(), _cfg(s, 64), 4)
    L = Light("directional", direction=np.array(light_dir))
    tau = fhv.shadow_transmittance(pa, np.array([0.5, 0.5, 0.2]), L, fhv.default_raycast_config(pa))
    assert abs(tau - expect) <= 1e-6


def _slab_np(o, d, lo, hi):
    """Brute-force ray / AABB over [0, inf) for many boxes (the reference's
    _slab semantics, fhv/raycast.py:179-202)."""
    t0 = np.zeros(len(lo))
    t1 = np.full(len(lo), np.inf)
    ok = np.ones(len(lo), bool)
    for a in range(3):
        if d[a] == 0.0:
            ok &= ~((o[a] < lo[:, a]) | (o[a] > hi[:, a]))
        else:
            ta, tb = (lo[:, a] - o[a]) / d[a], (hi[:, a] - o[a]) / d[a]
            t0 = np.maximum(t0, np.minimum(ta, tb))
            t1 = np.minimum(t1, np.maximum(ta, tb))
    return ok & (t0 <= t1)


@pytest.mark.parametrize("L", [2, 3, 4])
def test_12_traversal_order_and_completeness(L):
    rng = np.random.default_rng(12 + L)
    occ = rng.random(8 ** L) < 0.08
    pyr = fhv.OccupancyPyramid.from_leaf_occupancy(occ, L)
    codes = np.flatnonzero(occ)
    ijk = np.stack(fhv.morton_decode(codes, L), axis=1).astype(np.float64)
    size = 1.0 / (1 << L)
    lo, hi = ijk * size, ijk * size + size
    n_rays = 10_000 if L == 4 else 2_000
    for _ in range(n_rays):
        o = rng.uniform(-0.5, 1.5, 3)
        d = rng.normal(size=3)
        if rng.random() < 0.1:
            d[rng.integers(3)] = 0.0  # axis-parallel rays exercise the d = 0 slab branch
        if not d.any():
            continue
        ray = fhv.Ray(o, d)
        seq = []
        fhv.traverse_octree(pyr, ray, lambda c, te, tx: seq.append((c, te)) or True)
        visited = [c for c, _ in seq]
        te = [t for _, t in seq]
        assert all(a <= b for a, b in zip(te, te[1:]))
        expect = set(codes[_slab_np(ray.origin, ray.direction, lo, hi)].tolist())
        assert expect <= set(visited)
        assert set(visited) <= set(codes.tolist())


def test_traversal_examples():
    # leaves along +x visited in ascending x; a ray pointing away and an empty pyramid -> 0
    L = 2
    occ = np.zeros(8 ** L, bool)
    codes = [fhv.morton_encode(x, 1, 2, L) for x in range(4)]
    occ[codes] = True
    pyr = fhv.OccupancyPyramid.from_leaf_occupancy(occ, L)
    seq = []
    fhv.traverse_octree(pyr, fhv.Ray(np.array([-1.0, 0.3, 0.6]), np.array([1.0, 0.0, 0.0])),
                        lambda c, a, b: seq.append(c) or True)
    assert seq == codes
    assert fhv.traverse_octree(pyr, fhv.Ray(np.array([2.0, 0.3, 0.6]), np.array([1.0, 0.0, 0.0])),
                               lambda *a: True) == 0
    empty = fhv.OccupancyPyramid(L)
    assert fhv.traverse_octree(empty, fhv.Ray(np.array([-1.0, 0.3, 0.6]), np.array([1.0, 0.0, 0.0])),
                               lambda *a: True) == 0
    # intersect_fragment examples
    r = fhv.Ray(np.zeros(3), np.array([1.0, 0.0, 0.0]))
    assert fhv.intersect_fragment(r, (5.0, 0.0, 0.0), 0.1) == 5.0
    assert fhv.intersect_fragment(r, (5.0, 0.2, 0.0), 0.1) is None
    assert fhv.intersect_fragment(r, (-1.0, 0.0, 0.0), 0.1) is None
