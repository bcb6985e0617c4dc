"""GPU parity of the reference's per-call / scalar API against the reference's
own outputs (tests/golden/scalar.npz, tests/golden/make_golden_scalar.py):

* kernels() operator module: coverage, linked_insert, pofa_scatter bit-exact
  (NumPy arguments and CUDA tensors), raycast_image == render_raycast;
* rasterize_triangle (orthographic + perspective) and capture_pass depth:
  pixels, f64 positions / normals / depth bit-exact;
* traverse_octree / gather_ray_hits / intersect_fragment / project_points /
  shade_many bit-exact; raycast_pixel hits and stats exact, colours within
  TOL = 1e-12 (the reference's Python scalar path shades with np.dot --
  BLAS FMA chains -- where its compiled kernel and this device use plain
  products; same for shadow_transmittance's light distance);
* ppfl_insert / pofl_insert / set_paths / from_leaf_occupancy / chain_indices
  bit-exact, including pool overflow (None) semantics.
"""
import numpy as np
import pytest
import torch

import paper_2211_15460_b200 as fhv
from paper_2211_15460_b200 import kernels, raycast, render, storage
from paper_2211_15460_b200.lights import Light
from paper_2211_15460_b200.raster import CaptureStrategy as CS
from paper_2211_15460_b200.raster import RasterConfig
from paper_2211_15460_b200.scene import capture_camera, viewpoint_camera
from tests._golden import golden_scene, npz

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module")
def g():
    return npz("scalar")


# ---- operator module --------------------------------------------------------

def test_coverage_bit_exact(g):
    w, h = (int(v) for v in g["cov/wh"])
    for i, t in enumerate(g["cov/tris"]):
        px, py, l0, l1, l2 = kernels.coverage(*[float(v) for v in t], w, h)
        assert px.dtype == np.int32 and l0.dtype == np.float64
        assert np.array_equal(px, g[f"cov/{i}/px"]) and np.array_equal(py, g[f"cov/{i}/py"])
        assert np.array_equal(np.stack([l0, l1, l2], 1).reshape(-1, 3), g[f"cov/{i}/l"].reshape(-1, 3))
    with pytest.raises(ValueError):
        kernels.coverage(0.0, 0.0, 0.0, 10.0, 10.0, 0.0, w, h)
    # one batched launch pair == the per-triangle calls, concatenated
    n = len(g["cov/tris"])
    r = kernels.coverage_batch(g["cov/tris"], np.tile(g["cov/wh"], (n, 1)))
    assert r["first_bad"] == -1
    off = r["tri_off"].cpu().numpy()
    assert np.array_equal(np.diff(off), [len(g[f"cov/{i}/px"]) for i in range(n)])
    assert np.array_equal(r["px"].cpu().numpy(), np.concatenate([g[f"cov/{i}/px"] for i in range(n)]))
    lam = np.concatenate([g[f"cov/{i}/l"].reshape(-1, 3) for i in range(n)])
    assert np.array_equal(r["l2"].cpu().numpy(), lam[:, 2])


def test_coverage_large_triangle_matches_oracle():
    from oracle import oracle as orc
    t = (3.25, -40.0, 1500.5, 700.0, -9.0, 1300.75)
    px, py, l0, l1, l2 = kernels.coverage(*t, 1280, 1024)
    opx, opy, lam = orc.coverage(*t, 1280, 1024)
    assert len(px) > 500_000
    assert np.array_equal(px, opx) and np.array_equal(py, opy)
    assert np.array_equal(np.stack([l0, l1, l2], 1), lam)


@pytest.mark.parametrize("where", ["numpy", "cuda"])
def test_linked_insert_bit_exact(g, where):
    heads = np.full(50, -1, np.int32)
    heads[:10] = np.arange(10, dtype=np.int32)
    prev = np.full(400, -7, np.int32)
    if where == "cuda":
        th, tp = torch.from_numpy(heads).cuda(), torch.from_numpy(prev).cuda()
        kernels.linked_insert(torch.from_numpy(g["li/keys"]).cuda(), th, tp, 40)
        heads, prev = th.cpu().numpy(), tp.cpu().numpy()
    else:
        kernels.linked_insert(g["li/keys"], heads, prev, 40)
    assert np.array_equal(heads, g["li/heads"]) and np.array_equal(prev, g["li/prev"])
    with pytest.raises(IndexError):
        kernels.linked_insert(np.array([3, 50]), heads, prev, 0)


@pytest.mark.parametrize("case", ["ok", "bad"])
@pytest.mark.parametrize("where", ["numpy", "cuda"])
def test_pofa_scatter_bit_exact(g, case, where):
    codes = g[f"ps/{case}/codes"]
    cur = np.zeros(40, np.uint32)
    dest = np.full(len(codes), -3, np.int64)
    if where == "cuda":
        tcur = torch.zeros(40, dtype=torch.int32, device="cuda").view(torch.uint32)
        tdest = torch.from_numpy(dest).cuda()
        bad = kernels.pofa_scatter(torch.from_numpy(codes).cuda(), torch.from_numpy(g["ps/offsets"].view(np.int32))
                                   .cuda().view(torch.uint32), torch.from_numpy(g["ps/counts"].view(np.int32)).cuda()
                                   .view(torch.uint32), tcur, tdest)
        cur = tcur.view(torch.int32).cpu().numpy().view(np.uint32)
        dest = tdest.cpu().numpy()
    else:
        bad = kernels.pofa_scatter(codes, g["ps/offsets"], g["ps/counts"], cur, dest)
    assert bad == int(g[f"ps/{case}/bad"][0])
    assert np.array_equal(cur, g[f"ps/{case}/cursors"]) and np.array_equal(dest, g[f"ps/{case}/dest"])


def test_raycast_image_operator_matches_render_raycast():
    s = golden_scene("cornell")
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 64))
    pa = fhv.pofa_build(s, CS.three_way_geometry(), cfg, 5)
    cam = viewpoint_camera("+z", (40, 24), "perspective", 45.0, 1.2)
    lights = [fhv.headlight(cam)]
    rc = fhv.default_raycast_config(pa, mode="transparency_shadows")
    bg = (0.1, 0.2, 0.3, 0.5)
    img, st, ids = fhv.render_raycast(pa, cam, lights, rc, background=bg, collect_ids=True)
    o, d = fhv.primary_rays(cam)
    mats = fhv.lights.material_arrays(s.materials)
    from paper_2211_15460_b200.lights import pack_lights
    lk, lv, lc, la = pack_lights(lights)
    pool = pa.pool.numpy()
    L = pa.levels
    pyr = pa.pyramid.data.cpu().numpy()
    pyr_off = np.array([((1 << (3 * k)) - 1) // 7 for k in range(L)], np.int64)
    out = np.empty((40 * 24, 4))
    out[:] = bg
    out_ids = np.full(40 * 24, -1, np.int32)
    counters = np.zeros(4, np.int64)
    for r0, r1 in ((0, 10), (10, 24)):  # two spans, like the reference's row chunks
        kernels.raycast_image(r0 * 40, r1 * 40, o, d, 0, L, pa.directory.offsets.cpu().numpy().astype(np.int64),
                              pa.directory.counts.cpu().numpy().astype(np.int64), pyr, pyr_off, pool["position"],
                              pool["normal"], pool["material_id"].astype(np.int64),
                              pool["object_id"].astype(np.int64), mats["diffuse"], mats["specular"],
                              mats["shininess"], mats["alpha"], lk, lv, lc, la, cam.eye, np.array(bg), rc.splat_radius_world,
                              1.0, 2, rc.shadow_epsilon, out, out_ids, counters)
    assert np.array_equal(out.reshape(24, 40, 4), img.pixels.cpu().numpy())
    assert np.array_equal(out_ids.reshape(24, 40), ids.cpu().numpy())
    assert list(counters) == list(st.as_dict().values())


# ---- rasterize_triangle / capture_pass depth --------------------------------

@pytest.mark.parametrize("cname", ["ortho", "persp"])
def test_rasterize_triangle_bit_exact(g, cname):
    s = golden_scene("icosphere")
    cam = viewpoint_camera("+y", (48, 40), "orthographic") if cname == "ortho" else \
        viewpoint_camera("+x", (48, 40), "perspective", 50.0, 1.3)
    cfg = RasterConfig.from_camera(cam)
    assert np.array_equal(cfg.projection, g[f"rt/{cname}/proj"])
    out = fhv.rasterize_triangles(s, cfg)
    k = f"rt/{cname}/"
    assert np.array_equal(out["job"].cpu().numpy(), g[k + "tri"])
    for name, key in (("raster_x", "px"), ("raster_y", "py"), ("world_position", "pos"), ("world_normal", "nrm"),
                      ("depth", "depth")):
        assert np.array_equal(out[name].cpu().numpy(), g[k + key]), name
    # the per-triangle call and its sink
    cnt = g[k + "count"]
    for t in (0, 7, int(np.argmax(cnt))):
        sink = fhv.ListSink()
        n = fhv.rasterize_triangle(s.triangles[t], cfg, sink)
        assert n == cnt[t]
        sel = g[k + "tri"] == t
        if n:
            b = sink.batches[0]
            assert np.array_equal(b.world_position, g[k + "pos"][sel]) and np.array_equal(b.depth, g[k + "depth"][sel])
            f = next(b.fragments())
            assert f.raster_xy == (int(g[k + "px"][sel][0]), int(g[k + "py"][sel][0]))
        else:
            assert not sink.batches


@pytest.mark.parametrize("st", ["one_view", "three_separate", "three_way_geometry", "normal_space"])
def test_capture_pass_depth_bit_exact(g, st):
    s = golden_scene("icosphere")
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 64))
    sink = fhv.ListSink()
    fhv.capture_pass(s, CS(st), cfg, sink)
    assert np.array_equal([len(b) for b in sink.batches], g[f"cp/{st}/sizes"])
    assert np.array_equal(np.concatenate([b.depth for b in sink.batches]), g[f"cp/{st}/depth"])


# ---- ray queries --------------------------------------------------------------

@pytest.fixture(scope="module")
def vols():
    s = golden_scene("cornell")
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 64))
    return s, {"pofl": fhv.build_pofl(s, CS.three_way_geometry(), cfg, 5),
               "pofa": fhv.pofa_build(s, CS.three_way_geometry(), cfg, 5, exact_order=True)}


def _lights():
    return [Light("directional", direction=np.array([0.3, 0.5, 1.0]), ambient=(0.1, 0.1, 0.1)),
            Light("point", position=np.array([0.5, 0.9, 0.6]), color=(0.8, 0.7, 0.6))]


def _rays(g):
    out = []
    for i in range(int(g["ray/n"][0])):
        tt = g[f"ray/{i}/tt"]
        out.append(raycast.Ray(g[f"ray/{i}/o"], g[f"ray/{i}/d"], float(tt[0]), float(tt[1])))
    return out


def test_traverse_octree_bit_exact(g, vols):
    _, v = vols
    for i, r in enumerate(_rays(g)):
        seq = []
        n = fhv.traverse_octree(v["pofl"].pyramid, r, lambda c, a, b: seq.append((c, a, b)) or True)
        ref = g[f"ray/{i}/trav"]
        assert n == len(ref)
        assert np.array_equal(np.array(seq, dtype=np.float64).reshape(-1, 3), ref), i
        stop = []
        assert fhv.traverse_octree(v["pofl"].pyramid, r, lambda c, a, b: (stop.append(c), len(stop) < 3)[1]) == \
            int(g[f"ray/{i}/trav_stop3"][0])


@pytest.mark.parametrize("vname", ["pofl", "pofa"])
def test_gather_ray_hits_bit_exact(g, vols, vname):
    _, v = vols
    for i, r in enumerate(_rays(g)):
        st = fhv.RaycastStats()
        hits = raycast.gather_ray_hits(v[vname], r, 1.0 / 64, st)
        got = np.array([(h.t, h.fragment_index, h.leaf) for h in hits], dtype=np.float64).reshape(-1, 3)
        assert np.array_equal(got, g[f"ray/{i}/{vname}/gather"]), i
        assert list(st.as_dict().values()) == list(g[f"ray/{i}/{vname}/gather_stats"])


@pytest.mark.parametrize("vname", ["pofl", "pofa"])
@pytest.mark.parametrize("mode", fhv.raycast.RAYCAST_MODES)
def test_raycast_pixel_matches_reference(g, vols, vname, mode):
    _, v = vols
    lights = _lights()
    for i, r in enumerate(_rays(g)):
        for cut in (1.0, 0.6, None):
            rc = fhv.default_raycast_config(v[vname], mode=mode, alpha_cutoff=cut)
            st = fhv.RaycastStats()
            ho = []
            rgba = fhv.raycast_pixel(v[vname], r, lights, rc, background=(0.1, 0.2, 0.3, 0.5), stats=st, hit_out=ho)
            k = f"ray/{i}/{vname}/{mode}/{cut}/"
            assert np.allclose(rgba, g[k + "rgba"], rtol=0, atol=TOL), (i, cut)
            assert list(st.as_dict().values()) == list(g[k + "stats"]), (i, cut)
            got = np.array([(h.t, h.fragment_index, h.leaf) for h in ho], dtype=np.float64).reshape(-1, 3)
            assert np.array_equal(got, g[k + "hits"]), (i, cut)


def test_shadow_transmittance_matches_reference(g, vols):
    _, v = vols
    pa = v["pofa"]
    rc = fhv.default_raycast_config(pa)
    pos = pa.pool.position.cpu().numpy()
    obj = pa.pool.object_id.cpu().numpy()
    for li, L in enumerate(_lights()):
        for ex in (0, 1):
            for j, i in enumerate(g["tau/sel"]):
                p = pos[i].astype(np.float64)
                code = int(storage.cell_code(p, pa.levels))
                st = fhv.RaycastStats()
                tau = fhv.shadow_transmittance(pa, p, L, rc, int(obj[i]) if ex else None, code if ex else None, st)
                assert abs(tau - g[f"tau/{li}/{ex}"][j]) <= TOL
                assert list(st.as_dict().values()) == list(g[f"tau/{li}/{ex}/stats"][j])


def test_intersect_fragment_bit_exact(g):
    rays = _rays(g)[:6]
    got = []
    for r in rays:
        for p in g["isect/pts"]:
            t = fhv.intersect_fragment(r, p, 0.15)
            got.append(np.nan if t is None else t)
    assert np.array_equal(np.array(got), g["isect/t"], equal_nan=True)


# ---- shading / projection -----------------------------------------------------

def test_shade_many_and_shade_bit_exact(g, vols):
    s, _ = vols
    lights = _lights()
    mats = fhv.lights.material_arrays(s.materials)
    P, N, M, eye = g["shade/P"], g["shade/N"], g["shade/M"], g["shade/eye"]
    assert np.array_equal(fhv.shade_many(P, N, M, mats, lights, eye), g["shade/many"])
    dev = fhv.shade_many(torch.from_numpy(P).cuda(), torch.from_numpy(N).cuda(), torch.from_numpy(M).cuda(),
                         s.materials, lights, eye)
    assert dev.is_cuda and np.array_equal(dev.cpu().numpy(), g["shade/many"])
    one = np.array([fhv.shade(P[i], N[i], s.materials[int(M[i])], lights[i % 2], eye) for i in range(8)])
    assert np.array_equal(one, g["shade/one"])


def test_project_points_bit_exact(g):
    cams = {"ortho": viewpoint_camera("+y", (40, 48), "orthographic"),
            "persp": viewpoint_camera("+z", (24, 16), "perspective", 45.0, 1.2)}
    P = g["shade/P"]
    for cname, cam in cams.items():
        xr, yr, d, zc = fhv.project_points(cam, P)
        assert np.array_equal(np.stack([xr, yr, d, zc], 1), g[f"proj/{cname}"])
        assert np.array_equal(np.array(fhv.project_points(cam, P[3])), g[f"proj/{cname}/one"])


# ---- single-fragment inserts and pyramid helpers ------------------------------

def _frags(g):
    return [fhv.EmittedFragment((int(xy[0]), int(xy[1])), p, n, 0.5, int(mo[0]), int(mo[1]))
            for xy, p, n, mo in zip(g["ins/px"], g["ins/pos"], g["ins/nrm"], g["ins/mo"])]


def test_ppfl_insert_bit_exact(g):
    pool = fhv.FragmentPool(150)
    d = storage.PixelDirectory.empty(16, 16)
    idx = [fhv.ppfl_insert(d, pool, f) for f in _frags(g)]
    assert np.array_equal([-1 if v is None else v for v in idx], g["ins/ppfl_idx"])
    assert np.array_equal(d.heads.cpu().numpy(), g["ins/ppfl_heads"])
    assert np.array_equal(pool.prev_index.cpu().numpy(), g["ins/ppfl_prev"])
    assert [pool.next_free, int(pool.overflowed)] == list(g["ins/ppfl_nf"])
    with pytest.raises(fhv.FhvError):
        fhv.ppfl_insert(d, pool, fhv.EmittedFragment((16, 0), np.zeros(3), np.zeros(3), 0.5, 0, 0))


def test_pofl_insert_pyramid_chains_bit_exact(g):
    pool = fhv.FragmentPool(250)
    d = storage.PoflDirectory.empty(3)
    pyr = fhv.OccupancyPyramid(3)
    idx = [fhv.pofl_insert(d, pyr, pool, f) for f in _frags(g)]
    assert np.array_equal(idx, g["ins/pofl_idx"])
    assert np.array_equal(d.heads.cpu().numpy(), g["ins/pofl_heads"])
    assert np.array_equal(pool.prev_index.cpu().numpy(), g["ins/pofl_prev"])
    assert np.array_equal(pyr.data.cpu().numpy(), g["ins/pofl_pyr"])
    assert np.array_equal(pool.position[:len(idx)].cpu().numpy(), g["ins/pofl_pos"])
    chains = [fhv.chain_indices(d.heads, pool.prev_index, int(k)) for k in g["ins/chain_keys"]]
    assert np.array_equal([len(c) for c in chains], g["ins/chain_len"])
    assert np.array_equal(np.concatenate(chains), g["ins/chain"])


def test_set_paths_and_from_leaf_occupancy_bit_exact(g):
    p = fhv.OccupancyPyramid(4)
    p.set_paths(g["sp/codes"])
    assert np.array_equal(p.data.cpu().numpy(), g["sp/pyr"])
    q = fhv.OccupancyPyramid.from_leaf_occupancy(g["occ/in"], 4)
    assert np.array_equal(q.data.cpu().numpy(), g["occ/pyr"])
    with pytest.raises(fhv.FhvError):
        p.set_paths(np.array([8 ** 4]))


def test_sinks_rebuild_the_bulk_builders():
    """capture_pass + the reference's sink objects == the fused device builders."""
    s = golden_scene("icosphere")
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 64))
    bulk = fhv.build_pofl(s, CS.normal_space(), cfg, 5, exact_order=True)
    pool = fhv.FragmentPool(bulk.pool.capacity)
    d = storage.PoflDirectory.empty(5)
    pyr = fhv.OccupancyPyramid(5)
    fhv.capture_pass(s, CS.normal_space(), cfg, fhv.PoflSink(d, pyr, pool))
    assert pool.next_free == bulk.pool.next_free
    assert torch.equal(d.heads, bulk.directory.heads) and torch.equal(pool.prev_index, bulk.pool.prev_index)
    assert torch.equal(pyr.data, bulk.pyramid.data)
    n = pool.next_free
    assert torch.equal(pool.position[:n], bulk.pool.position[:n]) and torch.equal(pool.normal[:n], bulk.pool.normal[:n])
    # two-pass POFA through CountingSink + PofaWriteSink
    pa = fhv.pofa_build(s, CS.normal_space(), cfg, 5, exact_order=True)
    cs = fhv.CountingSink(5)
    fhv.capture_pass(s, CS.normal_space(), cfg, cs)
    assert torch.equal(cs.counts, pa.directory.counts.view(torch.int32).to(torch.int64))
    pool = fhv.FragmentPool(pa.pool.capacity)
    ws = fhv.PofaWriteSink(pa.directory, pool)
    fhv.capture_pass(s, CS.normal_space(), cfg, ws)
    assert torch.equal(pool.position, pa.pool.position) and torch.equal(pool.normal, pa.pool.normal)
    assert torch.equal(ws.cursors.view(torch.int32), pa.directory.counts.view(torch.int32))
