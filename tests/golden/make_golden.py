"""Generate golden vectors by running the REFERENCE (`fhv`) in this container.

Usage:  python tests/golden/make_golden.py      (needs /root/reference)

The reference is copied to a scratch dir (it is read-only) and imported from
there.  Two backends are exercised:
  * "python"   -- the NumPy kernels, as shipped;
  * "compiled" -- the Cython kernels, built from the scratch copy with the
    five pointer casts SURVEY.md Appendix C describes (Cython 3.3 / NumPy 2
    reject `int64_t*` -> `long long*` at fhv/_ckern.pyx:676-683).  Built with
    `cython` + `gcc` directly (not the reference's setup.py).

Outputs (committed, small): tests/golden/*.npz plus golden_meta.json.  Big
arrays are stored as SHA-256 digests; small ones in full.  Nothing under
tests/ reads /root/reference at run time -- only this script does.
"""
from __future__ import annotations

import hashlib
import json
import os
import shutil
import subprocess
import sys
import sysconfig

import numpy as np

REF = "/root/reference/pkg/src"
SCRATCH = "/tmp/fhv_golden_ref"
OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def prepare_reference(compiled: bool):
    shutil.rmtree(SCRATCH, ignore_errors=True)
    shutil.copytree(REF, SCRATCH)
    for root, _, files in os.walk(SCRATCH):
        for f in files:
            os.chmod(os.path.join(root, f), 0o644)
    if compiled:
        pyx = os.path.join(SCRATCH, "fhv", "_ckern.pyx")
        src = open(pyx).read()
        for name in ("arr_a", "arr_b", "pyr_off", "pool_mat", "pool_obj"):
            src = src.replace(f"= &{name}[0]", f"= <long long*>&{name}[0]")
        open(pyx, "w").write(src)
        c_file = os.path.join(SCRATCH, "fhv", "_ckern.c")
        subprocess.run(["cython", "-3", pyx, "-o", c_file], check=True)
        inc = [sysconfig.get_paths()["include"], np.get_include()]
        so = os.path.join(SCRATCH, "fhv", "_ckern" + sysconfig.get_config_var("EXT_SUFFIX"))
        subprocess.run(["gcc", "-O3", "-shared", "-fPIC", "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION",
                        *[f"-I{i}" for i in inc], c_file, "-o", so, "-lm"], check=True)
    sys.path.insert(0, SCRATCH)


def scene_arrays(scene):
    T = len(scene.triangles)
    return {
        "positions": np.array([t.positions for t in scene.triangles]).reshape(T, 3, 3),
        "normals": np.array([t.normals for t in scene.triangles]).reshape(T, 3, 3),
        "face_normals": np.array([t.face_normal for t in scene.triangles]).reshape(T, 3),
        "material_id": np.array([t.material_id for t in scene.triangles], np.uint32),
        "object_id": np.array([t.object_id for t in scene.triangles], np.uint32),
        "mat_diffuse": np.array([m.diffuse for m in scene.materials], np.float64).reshape(-1, 3),
        "mat_specular": np.array([m.specular for m in scene.materials], np.float64).reshape(-1, 3),
        "mat_shininess": np.array([m.shininess for m in scene.materials], np.float64),
        "mat_alpha": np.array([m.alpha for m in scene.materials], np.float64),
    }


def cube972_reference(fhv_scene):
    """C1 scene built through the REFERENCE's make_triangle (same corner list
    as paper_2211_15460_b200.sample_scenes.cube972)."""
    Material, make_quad, Scene = fhv_scene.Material, fhv_scene.make_quad, fhv_scene.Scene
    mat = Material(diffuse=(0.7, 0.6, 0.5), specular=(0.2, 0.2, 0.2), shininess=32.0, alpha=1.0)
    lo, hi, n = 0.1, 0.9, 9
    g = [lo + (hi - lo) * i / n for i in range(n + 1)]
    faces = [(0, hi, 1, 2), (0, lo, 2, 1), (1, hi, 2, 0), (1, lo, 0, 2), (2, hi, 0, 1), (2, lo, 1, 0)]
    tris = []
    for obj, (ax, val, ua, va) in enumerate(faces):
        for i in range(n):
            for j in range(n):
                def P(a, b):
                    p = [0.0, 0.0, 0.0]
                    p[ax], p[ua], p[va] = val, g[a], g[b]
                    return tuple(p)
                tris += make_quad(P(i, j), P(i + 1, j), P(i + 1, j + 1), P(i, j + 1), 0, obj)
    return Scene.from_triangles(tris, [mat])


def pool_dict(pool, n, prefix, out, full):
    for k in ("position", "normal", "material_id", "object_id", "prev_index"):
        arr = np.ascontiguousarray(getattr(pool, k)[:n])
        if full:
            out[f"{prefix}{k}"] = arr
        out[f"{prefix}{k}_sha"] = np.array(sha(arr))


def main():
    backend = os.environ.get("GOLDEN_BACKEND", "compiled")
    prepare_reference(compiled=(backend == "compiled"))
    import fhv
    from fhv import sample_scenes, scene as fscene, raster, storage, render, raycast
    print("reference backend:", fhv.active_backend())
    meta = {"backend": fhv.active_backend(), "numpy": np.__version__}
    CS = raster.CaptureStrategy

    # ---- scenes and projections ------------------------------------------
    scenes = {name: sample_scenes.builtin_scene(name) for name in sample_scenes.builtin_names()}
    scenes["cube972"] = cube972_reference(fscene)
    sc_out = {}
    for name, s in scenes.items():
        for k, v in scene_arrays(s).items():
            sc_out[f"{name}/{k}"] = v
        for axis in ("+x", "+y", "+z"):
            for res in (32, 64, 256):
                cam = fscene.capture_camera(s, axis, res)
                sc_out[f"{name}/proj{axis}{res}"] = raster.RasterConfig.from_camera(cam).projection
    np.savez_compressed(os.path.join(OUT, "scenes.npz"), **sc_out)

    # ---- captures ----------------------------------------------------------
    cap = {}
    table = []
    for name in sample_scenes.builtin_names():
        s = scenes[name]
        for res in (32, 64, 256):
            cfg = raster.RasterConfig.from_camera(fscene.capture_camera(s, "+z", res))
            row = {"scene": name, "res": res}
            for st in ("one_view", "three_separate", "three_way_geometry", "normal_space"):
                sink = raster.ListSink()
                stats = raster.capture_pass(s, CS(st), cfg, sink)
                row[st] = stats.fragments_emitted
                key = f"{name}/{res}/list/{st}"
                if res <= 64 and sink.batches:
                    px = np.concatenate([b.raster_x for b in sink.batches]).astype(np.int32)
                    py = np.concatenate([b.raster_y for b in sink.batches]).astype(np.int32)
                    wp = np.concatenate([b.world_position for b in sink.batches])
                    wn = np.concatenate([b.world_normal for b in sink.batches])
                    cap[f"{key}/px_sha"] = np.array(sha(px))
                    cap[f"{key}/py_sha"] = np.array(sha(py))
                    cap[f"{key}/wpos_sha"] = np.array(sha(wp))
                    cap[f"{key}/wnrm_sha"] = np.array(sha(wn))
                cap[f"{key}/stats"] = np.array([stats.fragments_emitted, stats.triangles_processed,
                                                stats.passes, stats.draw_batches])
            v = storage.pofa_build(s, CS.normal_space(), cfg, 6)
            row["occupied_L6"] = int((v.directory.counts > 0).sum())
            row["counts_sha1_L6"] = hashlib.sha1(v.directory.counts.tobytes()).hexdigest()[:12]
            table.append(row)
            full = res == 32
            # PPFL one_view +z
            pp = storage.build_ppfl(s, cfg)
            k = f"{name}/{res}/ppfl/"
            pool_dict(pp.pool, pp.pool.stored_count, k, cap, full)
            cap[k + "heads_sha"] = np.array(sha(pp.directory.heads))
            if full:
                cap[k + "heads"] = pp.directory.heads
            cap[k + "meta"] = np.array([pp.pool.next_free, pp.pool.capacity, int(pp.pool.overflowed)])
            # PPFL with a tiny capacity (overflow semantics)
            small = max(1, pp.pool.next_free // 3)
            po = storage.build_ppfl(s, cfg, capacity=small)
            k = f"{name}/{res}/ppfl_small/"
            pool_dict(po.pool, po.pool.stored_count, k, cap, False)
            cap[k + "heads_sha"] = np.array(sha(po.directory.heads))
            cap[k + "meta"] = np.array([po.pool.next_free, po.pool.capacity, int(po.pool.overflowed)])
            for st, L in (("normal_space", 4), ("one_view", 4), ("three_way_geometry", 3)):
                pl = storage.build_pofl(s, CS(st), cfg, L)
                k = f"{name}/{res}/pofl_{st}_L{L}/"
                pool_dict(pl.pool, pl.pool.stored_count, k, cap, full)
                cap[k + "heads_sha"] = np.array(sha(pl.directory.heads))
                cap[k + "pyramid"] = np.concatenate(pl.pyramid.levels)
                cap[k + "meta"] = np.array([pl.pool.next_free, pl.pool.capacity, int(pl.pool.overflowed)])
                pa = storage.pofa_build(s, CS(st), cfg, L)
                k = f"{name}/{res}/pofa_{st}_L{L}/"
                pool_dict(pa.pool, pa.pool.stored_count, k, cap, full)
                cap[k + "offsets"] = pa.directory.offsets
                cap[k + "counts"] = pa.directory.counts
                cap[k + "pyramid"] = np.concatenate(pa.pyramid.levels)
                cap[k + "stats"] = np.array(list(pa.stats.as_dict().values()))
    np.savez_compressed(os.path.join(OUT, "captures.npz"), **cap)
    meta["appendix_b"] = table

    # ---- C1: cube972 @256 PPFL + splat ------------------------------------
    c1 = {}
    s = scenes["cube972"]
    cfg = raster.RasterConfig.from_camera(fscene.capture_camera(s, "+z", 256))
    pp = storage.build_ppfl(s, cfg)
    pool_dict(pp.pool, pp.pool.stored_count, "ppfl/", c1, False)
    c1["ppfl/heads_sha"] = np.array(sha(pp.directory.heads))
    c1["ppfl/meta"] = np.array([pp.pool.next_free, pp.pool.capacity, int(pp.pool.overflowed)])
    cam = fscene.viewpoint_camera("+x", (256, 256), "perspective")
    img = render.splat_render(pp.pool, cam, [render.headlight(cam)], 1.0 / 256, s.materials)
    c1["splat/rgba"] = img.pixels.astype(np.float32)
    c1["splat/rgba_sha"] = np.array(sha(img.pixels))
    c1["splat/depth_sha"] = np.array(sha(img.depth))
    np.savez_compressed(os.path.join(OUT, "c1.npz"), **c1)
    meta["c1_fragments"] = int(pp.pool.next_free)

    # ---- splat / raycast images on small captures -------------------------
    img_out = {}
    lights_sets = {
        "head": lambda cam: [render.headlight(cam)],
        "two": lambda cam: [render.Light("directional", direction=np.array([0.3, 0.8, 0.5]),
                                         color=(0.9, 0.8, 0.7), ambient=(0.05, 0.05, 0.05)),
                            render.Light("point", position=np.array([0.5, 1.4, 0.6]),
                                         color=(0.6, 0.6, 0.9), ambient=(0.02, 0.03, 0.04))],
    }
    cams = {
        "px_persp": fscene.viewpoint_camera("+x", (40, 32), "perspective"),
        "pz_ortho": fscene.viewpoint_camera("+z", (36, 36), "orthographic"),
        "py_persp": fscene.viewpoint_camera("+y", (32, 28), "perspective", fov_deg=50.0, distance=1.2),
    }
    for name in sample_scenes.builtin_names():
        s = scenes[name]
        cfg = raster.RasterConfig.from_camera(fscene.capture_camera(s, "+z", 32))
        pa = storage.pofa_build(s, CS.normal_space(), cfg, 4)
        pl = storage.build_pofl(s, CS.normal_space(), cfg, 4)
        pp = storage.build_ppfl(s, cfg)
        for cname, cam in cams.items():
            for lname, lf in lights_sets.items():
                lights = lf(cam)
                bg = (0.1, 0.2, 0.3, 0.5) if lname == "two" else (0.0, 0.0, 0.0, 0.0)
                for vname, vol in (("pofa", pa), ("ppfl", pp)):
                    gb = render.GBuffer.new(*cam.resolution)
                    im = render.splat_render(vol.pool, cam, lights, 1.0 / 32, s.materials, bg, gb)
                    k = f"{name}/splat/{vname}/{cname}/{lname}/"
                    img_out[k + "rgba"] = im.pixels
                    img_out[k + "depth"] = im.depth
                    img_out[k + "obj"] = gb.object_id
                if cname == "pz_ortho" and lname == "two":
                    continue
                for mode in ("opaque_nearest", "transparency", "transparency_shadows"):
                    rcfg = raycast.default_raycast_config(pa, mode=mode)
                    for vname, vol in (("pofa", pa), ("pofl", pl)):
                        im, st, ids = raycast.render_raycast(vol, cam, lights, rcfg, background=bg,
                                                             collect_ids=True)
                        k = f"{name}/ray/{vname}/{cname}/{lname}/{mode}/"
                        img_out[k + "rgba"] = im.pixels
                        img_out[k + "ids"] = ids
                        img_out[k + "stats"] = np.array(list(st.as_dict().values()))
                        img_out[k + "radius"] = np.array([rcfg.splat_radius_world, rcfg.shadow_epsilon])
    np.savez_compressed(os.path.join(OUT, "images.npz"), **img_out)

    # ---- closed forms ------------------------------------------------------
    s = scenes["three-quads"]
    cfg = raster.RasterConfig.from_camera(fscene.capture_camera(s, "+z", 64))
    pa = storage.pofa_build(s, CS.normal_space(), cfg, 4)
    light = render.Light("directional", direction=np.array([0.0, 0.0, 1.0]))
    rcfg = raycast.default_raycast_config(pa)
    ray = raycast.Ray(np.array([0.45, 0.55, 1.5]), np.array([0.0, 0.0, -1.0]))
    rgba = raycast.raycast_pixel(pa, ray, [light], rcfg, background=(0, 0, 0, 0))
    meta["fig2_rgba"] = [float(x) for x in rgba]
    tau = raycast.shadow_transmittance(pa, np.array([0.5, 0.5, 0.05]), light, rcfg)
    meta["shadow_tau_3quads"] = float(tau)
    meta["memory"] = {
        "ppfl_1000": storage.memory_report("PPFL", resolution=(1000, 1000)),
        "pofl_1000": [storage.memory_report("POFL", resolution=(1000, 1000), levels=L)["total_bytes"] for L in (6, 7, 8)],
        "pofa_0": [storage.memory_report("POFA", levels=L, exact_count=0)["total_bytes"] for L in (6, 7, 8)],
    }
    json.dump(meta, open(os.path.join(OUT, "golden_meta.json"), "w"), indent=1, default=str)
    print("wrote goldens to", OUT)


if __name__ == "__main__":
    main()
