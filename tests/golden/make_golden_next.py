"""Golden vectors for the SURVEY.md section 8(f) rows, made by running the
REFERENCE (`fhv`) in this container (same scratch-copy recipe and compiled
backend as make_golden.py):

  * deferred_baseline (fhv/render.py:327-382): image rgba / depth and the full
    G-buffer for every built-in scene x {perspective, orthographic} cameras x
    two light sets (and a background);
  * FHV1 snapshots (fhv/storage.py:725-808): SHA-256 of snapshot_bytes for
    PPFL / POFL / POFA volumes of each built-in at 32^2 (+ the full bytes of
    the smallest);
  * rebuild_pofl_as_pofa (fhv/storage.py:624-652): directory + pool.

Usage:  python tests/golden/make_golden_next.py      (needs /root/reference)
Output: tests/golden/next.npz (committed).
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import OUT, prepare_reference, sha  # noqa: E402


def near_camera(Camera):
    """Perspective camera INSIDE the unit cube: some triangles have clip w <= 1e-9
    (behind the eye) and are skipped by _raster_screen (fhv/raster.py:189-190)."""
    return Camera("perspective", np.array([0.5, 0.45, 0.62]), np.array([0.1, 0.05, -1.0]), np.array([0.0, 1.0, 0.0]),
                  75.0, (48, 40), 0.01, 2.0)


def main():
    prepare_reference(compiled=os.environ.get("GOLDEN_BACKEND", "compiled") == "compiled")
    import fhv
    from fhv import raster, render, sample_scenes, scene as fscene, storage
    print("reference backend:", fhv.active_backend())
    CS = raster.CaptureStrategy
    out = {}
    cams = {
        "px_persp": fscene.viewpoint_camera("+x", (40, 32), "perspective"),
        "pz_ortho": fscene.viewpoint_camera("+z", (36, 36), "orthographic"),
        "py_persp": fscene.viewpoint_camera("+y", (32, 28), "perspective", fov_deg=50.0, distance=1.2),
        "near_persp": near_camera(fscene.Camera),
    }
    lights_sets = {
        "head": lambda cam: [render.headlight(cam)],
        "two": lambda cam: [render.Light("directional", direction=np.array([0.3, 0.8, 0.5]),
                                         color=(0.9, 0.8, 0.7), ambient=(0.05, 0.05, 0.05)),
                            render.Light("point", position=np.array([0.5, 1.4, 0.6]),
                                         color=(0.6, 0.6, 0.9), ambient=(0.02, 0.03, 0.04))],
    }
    for name in sample_scenes.builtin_names():
        s = sample_scenes.builtin_scene(name)
        for cname, cam in cams.items():
            for lname, lf in lights_sets.items():
                bg = (0.1, 0.2, 0.3, 0.5) if lname == "two" else (0.0, 0.0, 0.0, 0.0)
                img, gb = render.deferred_baseline(s, cam, lf(cam), bg)
                k = f"{name}/deferred/{cname}/{lname}/"
                out[k + "rgba"] = img.pixels
                out[k + "depth"] = img.depth
                out[k + "gpos"] = gb.position
                out[k + "gnrm"] = gb.normal
                out[k + "gmat"] = gb.material_id
                out[k + "gobj"] = gb.object_id
                out[k + "valid"] = gb.valid
        cfg = raster.RasterConfig.from_camera(fscene.capture_camera(s, "+z", 32))
        pp = storage.build_ppfl(s, cfg)
        pl = storage.build_pofl(s, CS.normal_space(), cfg, 4)
        pa = storage.pofa_build(s, CS.normal_space(), cfg, 4)
        for vname, vol in (("ppfl", pp), ("pofl", pl), ("pofa", pa)):
            blob = storage.snapshot_bytes(vol)
            out[f"{name}/snapshot/{vname}/sha"] = np.array(sha(np.frombuffer(blob, np.uint8)))
            out[f"{name}/snapshot/{vname}/len"] = np.array(len(blob))
            if name == "three-quads" and vname == "pofa":
                out[f"{name}/snapshot/{vname}/bytes"] = np.frombuffer(blob, np.uint8)
        for st, L in (("normal_space", 4), ("three_way_geometry", 3)):
            pl = storage.build_pofl(s, CS(st), cfg, L)
            rb = storage.rebuild_pofl_as_pofa(pl)
            k = f"{name}/rebuild/{st}_L{L}/"
            out[k + "offsets"] = rb.directory.offsets
            out[k + "counts"] = rb.directory.counts
            out[k + "pyramid"] = np.concatenate(rb.pyramid.levels)
            n = rb.pool.stored_count
            for f in ("position", "normal", "material_id", "object_id", "prev_index"):
                out[k + f + "_sha"] = np.array(sha(getattr(rb.pool, f)[:n]))
            out[k + "n"] = np.array(n)
    np.savez_compressed(os.path.join(OUT, "next.npz"), **out)
    print("wrote", os.path.join(OUT, "next.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
