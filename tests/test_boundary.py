"""CPU-side checks of the drop-in boundary and host logic (no GPU needed)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2211_15460_b200 as fhv
from paper_2211_15460_b200 import _lib, sample_scenes
from paper_2211_15460_b200.raster import CaptureStrategy, RasterConfig, capture_plan
from paper_2211_15460_b200.scene import capture_camera
from tests._golden import meta

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "fhv_b200.h")).read()
    return sorted(set(re.findall(r"\b(fhv_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load(require_cuda=False)
    names = _header_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTED)
    assert lib.fhv_version().startswith(b"fhv_b200")


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.Tris) == 48
    assert ctypes.sizeof(_lib.CaptureCfg) == 8 + 8 + 48 * 8
    assert ctypes.sizeof(_lib.Pool) == 48
    assert ctypes.sizeof(_lib.Shading) == 80
    assert ctypes.sizeof(_lib.Volume) == 80


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    s = sample_scenes.overlap_quads()
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 32))
    with pytest.raises(RuntimeError):
        fhv.pofa_build(s, CaptureStrategy.normal_space(), cfg, 4)


def test_morton_roundtrip_exhaustive():
    """SPEC acceptance 1: decode(encode) identity for L = 1..7 over all codes."""
    for L in range(1, 8):
        codes = np.arange(8 ** L, dtype=np.int64)
        x, y, z = fhv.morton_decode(codes, L)
        assert np.array_equal(fhv.morton_encode(x, y, z, L), codes)
    assert fhv.morton_encode(1, 1, 1, 1) == 7
    assert fhv.morton_encode(1, 0, 1, 1) == 5
    assert tuple(fhv.cell_of((0.999, 0.5, 0.25), 2)) == (3, 2, 1)


def test_memory_report_matches_reference():
    m = meta()["memory"]
    assert fhv.memory_report("PPFL", resolution=(1000, 1000))["total_bytes"] == m["ppfl_1000"]["total_bytes"]
    assert [fhv.memory_report("POFL", resolution=(1000, 1000), levels=L)["total_bytes"] for L in (6, 7, 8)] == m["pofl_1000"]
    assert [fhv.memory_report("POFA", levels=L, exact_count=0)["total_bytes"] for L in (6, 7, 8)] == m["pofa_0"]


def test_capture_plan_job_mapping():
    s = sample_scenes.cornell_box()
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 64))
    for kind, jobs, passes in (("one_view", 34, 1), ("three_separate", 102, 3), ("three_way_geometry", 102, 1),
                               ("normal_space", 34, 1)):
        p = capture_plan(s, CaptureStrategy(kind), cfg)
        assert (p.n_jobs, p.passes) == (jobs, passes)
        assert p.stats(0).draw_batches == passes * 7
    p = capture_plan(s, CaptureStrategy.normal_space(), cfg)
    assert p.pitch == 1.0 / 64


def test_sphere_field_matches_per_triangle_make_triangle():
    """The struct-of-arrays bench builder reproduces make_triangle bit for bit."""
    s = sample_scenes.sphere_field(2, 2, seed=7, r_lo=0.05, r_hi=0.2, c_lo=0.3, c_hi=0.7)
    verts, faces = sample_scenes.icosphere_mesh(2)
    rng = np.random.default_rng(7)
    centers = rng.uniform(0.3, 0.7, size=(2, 3))
    radii = rng.uniform(0.05, 0.2, size=2)
    k = 0
    for sp in range(2):
        for a, b, c in faces:
            t = fhv.make_triangle(centers[sp] + radii[sp] * verts[a], centers[sp] + radii[sp] * verts[b],
                                  centers[sp] + radii[sp] * verts[c], verts[a], verts[b], verts[c])
            assert np.array_equal(t.positions, s.positions[k])
            assert np.array_equal(t.normals, s.normals[k])
            assert np.array_equal(t.face_normal, s.face_normals[k])
            k += 1
