"""GPU parity for the SURVEY.md section 8(f) rows against the reference's own
outputs (tests/golden/next.npz) and the CPU oracle:

* deferred_baseline on the device: depth, G-buffer (f64 position / normal,
  ids, valid) bit-exact; colours within TOL = 1e-12 (CUDA pow vs libm pow);
* FHV1 snapshots written from device buffers: byte-identical (SHA-256) to the
  reference's snapshot_bytes for PPFL / POFL / POFA; load -> save round trip;
* rebuild_pofl_as_pofa on the device: directory, pyramid and every record
  byte bit-exact; equal to a direct pofa_build of the same capture.
"""
import os
import tempfile

import numpy as np
import pytest
import torch

import paper_2211_15460_b200 as fhv
from oracle import oracle as orc
from paper_2211_15460_b200.raster import CaptureStrategy, RasterConfig
from paper_2211_15460_b200.scene import capture_camera
from tests._golden import BUILTINS, golden_scene, npz, sha
from tests.test_next_oracle import CAMS, TOL, background, lights_for

pytestmark = pytest.mark.gpu


def _np(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("name", BUILTINS)
@pytest.mark.parametrize("cname", sorted(CAMS))
@pytest.mark.parametrize("lname", ("head", "two"))
def test_deferred_matches_reference(name, cname, lname):
    s = golden_scene(name)
    cam = CAMS[cname]()
    img, gb = fhv.deferred_baseline(s, cam, lights_for(lname, cam), background(lname))
    g = npz("next")
    k = f"{name}/deferred/{cname}/{lname}/"
    assert gb.valid.dtype == torch.bool and gb.material_id.dtype == torch.int32
    assert np.array_equal(_np(img.depth), g[k + "depth"])
    for f, t in (("gpos", gb.position), ("gnrm", gb.normal), ("gmat", gb.material_id), ("gobj", gb.object_id),
                 ("valid", gb.valid)):
        assert np.array_equal(_np(t), g[k + f]), f
    np.testing.assert_allclose(_np(img.pixels), g[k + "rgba"], rtol=0, atol=TOL)


def test_deferred_matches_oracle_larger():
    """A bigger scene than the goldens (cube972, 1k triangles) at 256x192."""
    s = fhv.sample_scenes.cube972()
    cam = fhv.viewpoint_camera("+x", (256, 192), "perspective", fov_deg=55.0, distance=1.3)
    lights = lights_for("two", cam)
    img, gb = fhv.deferred_baseline(s, cam, lights, (0.1, 0.2, 0.3, 0.5))
    ref = orc.deferred(s, cam, lights, (0.1, 0.2, 0.3, 0.5))
    assert np.array_equal(_np(img.depth), ref["depth"])
    for f, t in (("gpos", gb.position), ("gnrm", gb.normal), ("gmat", gb.material_id), ("gobj", gb.object_id),
                 ("valid", gb.valid)):
        assert np.array_equal(_np(t), ref[f]), f
    np.testing.assert_allclose(_np(img.pixels), ref["rgba"], rtol=0, atol=TOL)


def _vols(s):
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 32))
    ns = CaptureStrategy.normal_space()
    return {"ppfl": fhv.build_ppfl(s, cfg, exact_order=True),
            "pofl": fhv.build_pofl(s, ns, cfg, 4, exact_order=True),
            "pofa": fhv.pofa_build(s, ns, cfg, 4, exact_order=True)}


@pytest.mark.parametrize("name", BUILTINS)
def test_snapshot_bytes_match_reference(name):
    s = golden_scene(name)
    g = npz("next")
    for vname, vol in _vols(s).items():
        blob = fhv.snapshot_bytes(vol)
        assert len(blob) == int(g[f"{name}/snapshot/{vname}/len"]), vname
        assert sha(np.frombuffer(blob, np.uint8)) == str(g[f"{name}/snapshot/{vname}/sha"]), vname


@pytest.mark.parametrize("name", BUILTINS)
def test_snapshot_round_trip(name):
    s = golden_scene(name)
    with tempfile.TemporaryDirectory() as d:
        for vname, vol in _vols(s).items():
            path = os.path.join(d, vname + ".fhv")
            fhv.save_snapshot(vol, path)
            back = fhv.load_snapshot(path, materials=s.materials)
            assert back.layout == vol.layout
            assert fhv.snapshot_bytes(back) == open(path, "rb").read()


def test_load_reference_snapshot_bytes():
    """The reference's own bytes (three-quads POFA L4) load and re-serialise identically."""
    blob = npz("next")["three-quads/snapshot/pofa/bytes"].tobytes()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "ref.fhv")
        open(path, "wb").write(blob)
        vol = fhv.load_snapshot(path)
        assert vol.layout == "POFA" and vol.levels == 4
        assert fhv.snapshot_bytes(vol) == blob


def test_snapshot_errors():
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "bad.fhv")
        open(path, "wb").write(b"FHV")
        with pytest.raises(fhv.FhvError):
            fhv.load_snapshot(path)
        open(path, "wb").write(b"XXXX" + bytes(28))
        with pytest.raises(fhv.FhvError):
            fhv.load_snapshot(path)


@pytest.mark.parametrize("name", BUILTINS)
@pytest.mark.parametrize("st,L", (("normal_space", 4), ("three_way_geometry", 3)))
def test_rebuild_pofl_as_pofa_matches_reference(name, st, L):
    s = golden_scene(name)
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 32))
    # any POFL pool order gives the same repack only up to in-leaf order; the
    # reference repacks its own (sequential) pool, so rebuild from the exact one
    pl = fhv.build_pofl(s, CaptureStrategy(st), cfg, L, exact_order=True)
    rb = fhv.rebuild_pofl_as_pofa(pl)
    g = npz("next")
    k = f"{name}/rebuild/{st}_L{L}/"
    assert rb.pool.stored_count == int(g[k + "n"])
    assert np.array_equal(_np(rb.directory.offsets), g[k + "offsets"])
    assert np.array_equal(_np(rb.directory.counts), g[k + "counts"])
    assert np.array_equal(_np(rb.pyramid.data), g[k + "pyramid"])
    h = rb.pool.numpy()
    for f in ("position", "normal", "material_id", "object_id", "prev_index"):
        assert sha(h[f]) == str(g[k + f + "_sha"]), f


def test_rebuild_equals_direct_pofa_build():
    """rebuild(POFL) == pofa_build of the same capture (the cross-layout oracle, fhv/storage.py:627-630)."""
    s = fhv.sample_scenes.cube972()
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 256))
    ns = CaptureStrategy.normal_space()
    rb = fhv.rebuild_pofl_as_pofa(fhv.build_pofl(s, ns, cfg, 6, exact_order=True))
    pa = fhv.pofa_build(s, ns, cfg, 6, exact_order=True)
    assert torch.equal(rb.directory.offsets, pa.directory.offsets)
    assert torch.equal(rb.directory.counts, pa.directory.counts)
    assert torch.equal(rb.pyramid.data, pa.pyramid.data)
    a, b = rb.pool.numpy(), pa.pool.numpy()
    for f in a:
        assert np.array_equal(a[f], b[f]), f


def _pool_from_positions(pos, dev):
    n = len(pos)
    pool = fhv.FragmentPool(n, dev)
    pool.position.copy_(torch.from_numpy(np.ascontiguousarray(pos, dtype=np.float32)))
    pool.normal.zero_()
    pool.material_id.zero_()
    pool.object_id.copy_(torch.arange(n, dtype=torch.int32, device=dev).view(torch.uint32))
    pool.next_free = n
    return pool


def test_device_cell_codes_on_adversarial_floats():
    """cell_code's f32 fast path (range bounds as floats, f32 floor) against the
    oracle's f64 restatement on floats straddling every leaf boundary and the
    [-1e-6, 1+1e-6] bounds, through the device repack's leaf histogram."""
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(7)
    vals = []
    for L in (8,):
        b = np.arange(0, 2 ** L + 1, dtype=np.float64) / 2 ** L
        f = b.astype(np.float32)
        for k in range(-3, 4):
            vals.append(f.view(np.int32) + k)
    edge = np.array([-1e-6, 1.0 + 1e-6, 0.0, 1.0], np.float32).view(np.int32)
    for k in range(-4, 5):
        vals.append(edge + k)
    v = np.concatenate(vals).view(np.float32)
    v = v[(v.astype(np.float64) >= -1e-6) & (v.astype(np.float64) <= 1.0 + 1e-6)]
    pos = np.stack([rng.permutation(v), rng.permutation(v), rng.permutation(v)], axis=1).astype(np.float32)
    L = 8
    codes = orc.cell_codes(pos, L)
    vol = fhv.FhvPofl(fhv.storage.PoflDirectory(L, torch.full((8 ** L,), -1, dtype=torch.int32, device=dev)),
                      fhv.OccupancyPyramid(L, device=dev), _pool_from_positions(pos, dev), 256)
    rb = fhv.rebuild_pofl_as_pofa(vol)
    assert np.array_equal(rb.directory.counts.cpu().numpy(), np.bincount(codes, minlength=8 ** L).astype(np.uint32))
    for bad in (np.float32(np.nextafter(np.float32(-1e-6), np.float32(-1))), np.float32(1.0000011), np.float32("nan"),
                np.float32("inf")):
        p = pos[:4].copy()
        p[2, 1] = bad
        vol.pool = _pool_from_positions(p, dev)
        with pytest.raises(fhv.FhvError):
            fhv.rebuild_pofl_as_pofa(vol)
