"""Golden vectors for scene ingest, made by the
REFERENCE in this container: load_scene / load_material_table / save_scene /
normalize_scene (fhv/scene.py:251-487).

  * handcrafted files (fan polygons, missing normals, groups, usemtl switches,
    default material, -0.0, comments) and reference-saved built-in scenes:
    the file text + SHA-256 of every Scene array the reference loads, its
    materials, and normalize_scene's result;
  * error cases: the exact SceneLoadError message;
  * scatter1M (983,040 triangles) written by the reference's save_scene:
    SHA of the text and of the loaded arrays (the 1 M-triangle ingest case).

Usage:  python tests/golden/make_golden_ingest.py   (needs /root/reference; ~minutes)
Output: tests/golden/ingest_cases.json
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from make_golden import OUT, prepare_reference, scene_arrays, sha  # noqa: E402

MTL = """# name  kd(3) ks(3) shininess alpha
red 0.9 0.1 0.1 0.2 0.2 0.2 16 1
glass 0.6 0.7 0.8 0.5 0.5 0.5 64 0.25
"""

CASES = {
    "fan_polygons": ("""# quads and a pentagon, no normals, no groups
v 0 0 0
v 1 0 0
v 1 1 0
v 0 1 0
v 0.5 1.5 -0.0
v 0.25 0.5 0.75
f 1 2 3 4
f 1 2 5 3 4
f 1 2 6
""", None),
    "groups_materials": ("""v 0 0 0
v 1 0 0
v 0 1 0
v 0 0 1
vn 0 0 2
vn 1 1 1
vn -0.0 3 4
g left
usemtl red
f 1//1 2//2 3//3
g right
f 1//2 3//3 4//1
usemtl glass

f 2//3 3//1 4//2
g left
f 4 3 2
g
f 1 3 4
""", "mtl"),
    "default_material": ("""v 0.1 0.2 0.3
v 0.4 0.2 0.3
v 0.1 0.9 0.3
v 0.1 0.2 0.8
f 1 2 3
usemtl red
f 1 2 4
""", "mtl"),
    "degenerate": ("""v 0 0 0
v 1 1 1
v 2 2 2
vn 1e-150 0 0
f 1 2 3
f 1//1 2//1 3//1
""", None),
}

ERRORS = {
    "unknown_kw": "v 0 0 0\nvt 0 0\n",
    "v_count": "v 0 0\n",
    "v_float": "v 0 x 0\n",
    "v_nonfinite": "v 0 inf 0\n",
    "vn_zero": "v 0 0 0\nvn 0 0 0\n",
    "vn_tiny_zero": "vn 1e-200 -1e-170 1e-163\n",
    "face_short": "v 0 0 0\nf 1 1\n",
    "face_token": "v 0 0 0\nf 1/2/3 1 1\n",
    "face_token2": "v 0 0 0\nf 1/ 1 1\n",
    "face_int": "v 0 0 0\nf a 1 1\n",
    "face_range": "v 0 0 0\nf 1 2 1\n",
    "face_forward_ref": "v 0 0 0\nv 1 0 0\nf 1 2 3\nv 0 1 0\n",
    "normal_range": "v 0 0 0\nvn 0 0 1\nf 1//2 1//1 1//1\n",
    "usemtl_unknown": "usemtl nope\n",
    "usemtl_args": "usemtl\n",
    "empty": "# nothing\n\n",
    "first_error_wins": "v 0 0 0\nvn 0 0 0\nf 1 1\nbogus\n",
}

MTL_ERRORS = {
    "fields": "a 1 1 1 0 0 0 1\n",
    "float": "a 1 1 x 0 0 0 1 1\n",
    "nonfinite": "a 1 1 nan 0 0 0 1 1\n",
    "dup": "a 1 1 1 0 0 0 1 1\na 1 1 1 0 0 0 1 1\n",
    "range": "a 2 1 1 0 0 0 1 1\n",
    "shininess": "a 1 1 1 0 0 0 0 1\n",
}


def arrays_sha(scene):
    a = scene_arrays(scene)
    return {k: sha(v) for k, v in a.items()}


def main():
    prepare_reference(compiled=os.environ.get("GOLDEN_BACKEND", "compiled") == "compiled")
    from fhv import sample_scenes, scene as fscene
    meta = {"cases": {}, "errors": {}, "mtl_errors": {}, "saved": {}}
    npz = {}
    with tempfile.TemporaryDirectory() as d:
        mtl = os.path.join(d, "m.mtl")
        open(mtl, "w").write(MTL)
        for name, (text, m) in CASES.items():
            path = os.path.join(d, name + ".obj")
            open(path, "w").write(text)
            s = fscene.load_scene(path, mtl if m else None)
            ns, tr = fscene.normalize_scene(s, 0.05)
            meta["cases"][name] = {"text": text, "mtl": bool(m), "n": len(s.triangles),
                                   "arrays": arrays_sha(s), "materials": [
                                       [list(x.diffuse), list(x.specular), x.shininess, x.alpha] for x in s.materials],
                                   "norm_positions": sha(scene_arrays(ns)["positions"]),
                                   "scale": tr.scale, "offset": tr.offset.tolist()}
        meta["mtl_text"] = MTL
        for name, text in ERRORS.items():
            path = os.path.join(d, name + ".obj")
            open(path, "w").write(text)
            try:
                fscene.load_scene(path, mtl)
                raise SystemExit(f"{name}: no error")
            except fscene.SceneLoadError as e:
                meta["errors"][name] = {"text": text, "message": str(e).replace(path, "<path>"),
                                        "line": e.line_no}
        for name, text in MTL_ERRORS.items():
            path = os.path.join(d, name + ".mtl")
            open(path, "w").write(text)
            try:
                fscene.load_material_table(path)
                raise SystemExit(f"{name}: no error")
            except fscene.SceneLoadError as e:
                meta["mtl_errors"][name] = {"text": text, "message": str(e).replace(path, "<path>")}
        # reference-saved scenes: text + loaded arrays
        for name in sample_scenes.builtin_names() + ["scatter1m"]:
            if name == "scatter1m":
                sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
                from paper_2211_15460_b200 import sample_scenes as ours
                mine = ours.scatter1m()
                # the package's own scatter1M arrays as reference Triangles, verbatim
                tris = [fscene.Triangle(fscene.Vertex(p[0], n[0]), fscene.Vertex(p[1], n[1]),
                                        fscene.Vertex(p[2], n[2]), material_id=int(mi), object_id=int(oi),
                                        face_normal=f)
                        for p, n, f, mi, oi in zip(mine.positions, mine.normals, mine.face_normals,
                                                   mine.material_id, mine.object_id)]
                s = fscene.Scene.from_triangles(tris, [fscene.Material(m.diffuse, m.specular, m.shininess, m.alpha)
                                                       for m in mine.materials])
            else:
                s = sample_scenes.builtin_scene(name)
            obj, mp = os.path.join(d, name + ".obj"), os.path.join(d, name + ".mtl")
            fscene.save_scene(s, obj, mp)
            text = open(obj, "rb").read()
            back = fscene.load_scene(obj, mp)
            meta["saved"][name] = {"obj_sha": hashlib.sha256(text).hexdigest(), "obj_len": len(text),
                                   "mtl_sha": hashlib.sha256(open(mp, "rb").read()).hexdigest(),
                                   "n": len(back.triangles), "arrays": arrays_sha(back)}
            print(name, len(back.triangles), flush=True)
    json.dump(meta, open(os.path.join(OUT, "ingest_cases.json"), "w"), indent=1)
    print("wrote", os.path.join(OUT, "ingest_cases.json"))


if __name__ == "__main__":
    main()
