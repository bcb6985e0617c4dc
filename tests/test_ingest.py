"""Scene ingest against the reference's own
load_scene / load_material_table / save_scene / normalize_scene results
(tests/golden/ingest_cases.json, made by tests/golden/make_golden_ingest.py).

CPU: every error (SceneLoadError message with file:line, first error in file
order wins), material tables, the writer's exact text.  GPU: the loaded Scene
arrays bit-identical (normals are normalised on the device with the
reference's operation order), normalize_scene, and the 1 M-triangle scatter1M
round trip through the file format."""
import hashlib
import json
import os
import time

import numpy as np
import pytest

import paper_2211_15460_b200 as fhv
from paper_2211_15460_b200 import sample_scenes
from tests._golden import GOLDEN, sha

META = json.load(open(os.path.join(GOLDEN, "ingest_cases.json")))


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def _arrays_sha(s):
    return {"positions": sha(s.positions), "normals": sha(s.normals), "face_normals": sha(s.face_normals),
            "material_id": sha(s.material_id), "object_id": sha(s.object_id)}


@pytest.mark.parametrize("name", sorted(META["errors"]))
def test_load_errors_match_reference(tmp_path, name):
    case = META["errors"][name]
    mtl = _write(tmp_path, "m.mtl", META["mtl_text"])
    path = _write(tmp_path, name + ".obj", case["text"])
    with pytest.raises(fhv.SceneLoadError) as ei:
        fhv.load_scene(path, mtl)
    assert str(ei.value).replace(path, "<path>") == case["message"]
    assert ei.value.line_no == case["line"]


@pytest.mark.parametrize("name", sorted(META["mtl_errors"]))
def test_material_table_errors_match_reference(tmp_path, name):
    case = META["mtl_errors"][name]
    path = _write(tmp_path, name + ".mtl", case["text"])
    with pytest.raises(fhv.SceneLoadError) as ei:
        fhv.load_material_table(path)
    assert str(ei.value).replace(path, "<path>") == case["message"]


def test_material_table_loads(tmp_path):
    mats, names = fhv.load_material_table(_write(tmp_path, "m.mtl", META["mtl_text"]))
    assert names == {"red": 0, "glass": 1}
    assert mats[1].alpha == 0.25 and mats[0].diffuse == (0.9, 0.1, 0.1)


@pytest.mark.parametrize("name", ("cornell", "edge-plane", "icosphere", "three-quads"))
def test_save_scene_text_matches_reference(tmp_path, name):
    s = sample_scenes.builtin_scene(name)
    obj, mp = str(tmp_path / "s.obj"), str(tmp_path / "s.mtl")
    fhv.save_scene(s, obj, mp)
    want = META["saved"][name]
    assert hashlib.sha256(open(obj, "rb").read()).hexdigest() == want["obj_sha"]
    assert hashlib.sha256(open(mp, "rb").read()).hexdigest() == want["mtl_sha"]


def test_scene_transform():
    t = fhv.SceneTransform(2.0, np.array([0.5, 0.0, -1.0]))
    p = np.array([[1.0, 2.0, 3.0]])
    assert np.array_equal(t.invert(t.apply(p)), p)
    assert not t.is_identity and fhv.SceneTransform(1.0, np.zeros(3)).is_identity


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(META["cases"]))
def test_load_scene_matches_reference(tmp_path, name):
    case = META["cases"][name]
    mtl = _write(tmp_path, "m.mtl", META["mtl_text"]) if case["mtl"] else None
    s = fhv.load_scene(_write(tmp_path, name + ".obj", case["text"]), mtl)
    assert s.n_triangles == case["n"]
    got = _arrays_sha(s)
    assert got == {k: case["arrays"][k] for k in got}
    assert [[list(m.diffuse), list(m.specular), m.shininess, m.alpha] for m in s.materials] == case["materials"]
    ns, tr = fhv.normalize_scene(s, 0.05)
    assert sha(ns.positions) == case["norm_positions"]
    assert tr.scale == case["scale"] and tr.offset.tolist() == case["offset"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ("cornell", "edge-plane", "icosphere", "three-quads", "scatter1m"))
def test_save_load_round_trip_matches_reference(tmp_path, name):
    """Our writer produces the reference's text; our loader then yields the
    arrays the reference's loader yields from it (scatter1M: 983,040 faces)."""
    s = sample_scenes.scatter1m() if name == "scatter1m" else sample_scenes.builtin_scene(name)
    obj, mp = str(tmp_path / "s.obj"), str(tmp_path / "s.mtl")
    fhv.save_scene(s, obj, mp)
    want = META["saved"][name]
    assert hashlib.sha256(open(obj, "rb").read()).hexdigest() == want["obj_sha"]
    t0 = time.perf_counter()
    back = fhv.load_scene(obj, mp)
    dt = time.perf_counter() - t0
    assert back.n_triangles == want["n"]
    got = _arrays_sha(back)
    assert got == {k: want["arrays"][k] for k in got}
    if name == "scatter1m":
        print(f"load_scene scatter1M: {dt:.2f} s for {back.n_triangles} triangles")
