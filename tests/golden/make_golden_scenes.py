"""Golden vectors pinning the BIG bench scenes and their capture setup to the
REFERENCE (round 2; VERDICT r01 "scene pinning of the big configs").

  * scatter1M (C3/C5) and spheres100k (C2) built entirely by the reference:
    the same seeded draws (``np.random.default_rng(seed)``: centres, radii,
    colours), then one call of the reference's own ``icosphere(5, radius,
    centre)`` (fhv/sample_scenes.py:49-89, i.e. ``make_triangle`` per face)
    per sphere, material / object id = sphere index.  SHA-256 of positions,
    vertex normals, face normals and ids.
  * the capture setup of the 1920x1080 configs (C2-C5): ``capture_pass``'s
    pitch (``world_pixel_footprint``, fhv/raster.py:107-111) and the three
    axis projections ``ortho_projection(capture_camera(scene, axis, 1080))``
    (fhv/raster.py:37-51, fhv/scene.py:490-508), as exact float64 hex.
  * ingest: a ``vn`` whose squared norm overflows normalises to 0 and the
    reference raises ``SceneError("zero-length direction")`` from
    ``make_triangle`` at the first face using it, before a later bad line.

Usage:  python tests/golden/make_golden_scenes.py   (needs /root/reference; ~1 min)
Output: tests/golden/scenes_big.json
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import OUT, prepare_reference, scene_arrays, sha  # noqa: E402

# (n_spheres, subdivisions, seed, r_lo, r_hi, c_lo, c_hi, alpha): SURVEY.md 8(d) C2 / C3
RECIPES = {"spheres100k": (5, 5, 0, 0.05, 0.2, 0.2, 0.8, 0.6),
           "scatter1m": (48, 5, 1, 0.02, 0.12, 0.15, 0.85, 1.0)}

ZERO_VN = """v 0 0 0
v 1 0 0
v 0 1 0
vn 0 0 1
vn 1e200 0 0
f 1//1 2//1 3//1
f 1//2 2//1 3//1
bogus line
"""


def hexs(a) -> list:
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).reshape(-1)]


def main():
    prepare_reference(compiled=False)
    import fhv.sample_scenes as rss
    from fhv.raster import RasterConfig, ortho_projection, world_pixel_footprint
    from fhv.scene import Material, Scene, SceneError, capture_camera, load_scene
    out = {"scenes": {}}
    for name, (n, sub, seed, r_lo, r_hi, c_lo, c_hi, alpha) in RECIPES.items():
        rng = np.random.default_rng(seed)
        centers = rng.uniform(c_lo, c_hi, size=(n, 3))
        radii = rng.uniform(r_lo, r_hi, size=n)
        colors = rng.uniform(0.2, 0.9, size=(n, 3))  # per-sphere materials, drawn after the geometry
        tris = []
        for k in range(n):
            sph = rss.icosphere(sub, radius=float(radii[k]), center=centers[k], alpha=alpha)
            for t in sph.triangles:
                t.material_id = k
                t.object_id = k
            tris += sph.triangles
        mats = [Material(diffuse=tuple(float(c) for c in colors[k]), specular=(0.25, 0.25, 0.25), shininess=24.0,
                         alpha=alpha) for k in range(n)]
        scene = Scene.from_triangles(tris, mats)
        arr = scene_arrays(scene)
        cam = capture_camera(scene, "+z", 1080)
        cfg = RasterConfig((1920, 1080), RasterConfig.from_camera(cam).projection, extent=1.0)
        res = cfg.resolution[1]
        rec = {"n_triangles": len(tris),
               **{k + "_sha": sha(arr[k]) for k in ("positions", "normals", "face_normals", "material_id",
                                                    "object_id", "mat_diffuse", "mat_alpha")},
               "capture_res": res, "pitch": float(world_pixel_footprint(cfg)).hex(),
               "cfg_projection": hexs(cfg.projection),
               "axis_projection": {a: hexs(ortho_projection(capture_camera(scene, a, res)))
                                   for a in ("+x", "+y", "+z")}}
        out["scenes"][name] = rec
        print(name, rec["n_triangles"], rec["positions_sha"][:16])
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "z.obj")
        open(p, "w").write(ZERO_VN)
        try:
            load_scene(p)
            raise AssertionError("reference accepted a zero-length vertex normal")
        except SceneError as e:  # not a SceneLoadError: raised by make_triangle
            out["zero_vn"] = {"text": ZERO_VN, "type": type(e).__name__, "message": str(e)}
    json.dump(out, open(os.path.join(OUT, "scenes_big.json"), "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
