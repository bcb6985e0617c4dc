"""Python driver for the CPU oracle (liborc.so, built from fhv_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline and --impl reference).  It restates the reference's
capture / splat / ray-cast path sequentially in C (threads=1 semantics, the
reference's canonical order) and returns plain NumPy arrays shaped like the
reference's data structures.

Host-side setup that is not part of the hot path (projection matrices,
camera scalars, light packing) reuses the package's host helpers, which are
themselves pinned against the reference by tests/golden.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from paper_2211_15460_b200.lights import pack_lights, pack_materials
from paper_2211_15460_b200.raster import CaptureStrategy, capture_plan

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liborc.so")

OK, OVERFLOW, PASS_MISMATCH, BAD_ARGS, RANGE, BASIS, NOMEM, TOO_MANY, SPLAT_BIG = 0, 1, 2, 3, 5, 6, 7, 8, 9


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what} failed with status {code}")
        self.code = code


_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(
                os.path.join(HERE, "fhv_oracle.c")):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
    return _lib


class threads:
    """Context manager: run the oracle's POFA capture passes and splat on n
    host threads (CPU-baseline leg).  Directory, pyramid and splat image are
    unchanged; records inside a leaf land in a nondeterministic order."""

    def __init__(self, n: int):
        self.n = max(1, int(n))

    def __enter__(self):
        self.old = lib().orc_get_threads()
        lib().orc_set_threads(self.n)
        return self

    def __exit__(self, *exc):
        lib().orc_set_threads(self.old)


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _i64(v):
    return ctypes.c_int64(int(v))


def _f64(v):
    return ctypes.c_double(float(v))


def _tris(scene):
    return (np.ascontiguousarray(scene.positions), np.ascontiguousarray(scene.normals),
            np.ascontiguousarray(scene.face_normals), np.ascontiguousarray(scene.material_id),
            np.ascontiguousarray(scene.object_id))


def _plan_args(scene, strategy, cfg):
    plan = capture_plan(scene, strategy, cfg)
    proj = np.ascontiguousarray(plan.proj.reshape(3, 16))
    return plan, proj


def _stats(plan, raw):
    return plan.stats(int(raw[0])).as_dict()


def capture_list(scene, strategy, cfg, max_out=None):
    """Every fragment in emission order (ListSink, fhv/raster.py:309-320)."""
    plan, proj = _plan_args(scene, strategy, cfg)
    P, N, F, M, O = _tris(scene)
    raw = np.zeros(4, np.int64)
    n_out = np.zeros(1, np.int64)
    if max_out is None:
        dummy = np.zeros(1, np.int64)
        rc = lib().orc_capture_list(_i64(len(P)), _p(P), _p(N), _p(F), _p(M), _p(O), plan.strategy,
                                    plan.res, _f64(plan.pitch), _p(proj), 3, _i64(0), _p(dummy), None,
                                    None, None, None, None, None, _p(n_out), _p(raw))
        if rc:
            raise OracleError(rc, "capture_list")
        max_out = int(n_out[0])
    n = max_out
    job = np.zeros(n, np.int64)
    px = np.zeros(n, np.int32)
    py = np.zeros(n, np.int32)
    wpos = np.zeros((n, 3))
    wnrm = np.zeros((n, 3))
    mat = np.zeros(n, np.uint32)
    obj = np.zeros(n, np.uint32)
    rc = lib().orc_capture_list(_i64(len(P)), _p(P), _p(N), _p(F), _p(M), _p(O), plan.strategy,
                                plan.res, _f64(plan.pitch), _p(proj), 3, _i64(n), _p(job), _p(px),
                                _p(py), _p(wpos), _p(wnrm), _p(mat), _p(obj), _p(n_out), _p(raw))
    if rc:
        raise OracleError(rc, "capture_list")
    return {"job": job, "raster_x": px, "raster_y": py, "world_position": wpos,
            "world_normal": wnrm, "material_id": mat, "object_id": obj,
            "stats": _stats(plan, raw)}


def _touched(shape, dtype, fill=0):
    """np.full, i.e. pages faulted in here, once, rather than concurrently by
    the threaded passes (first-touch faults serialise on the mm lock)."""
    return np.full(shape, fill, dtype)


def _new_pool(cap):
    return {"position": _touched((cap, 3), np.float32), "normal": _touched((cap, 3), np.float32),
            "material_id": _touched(cap, np.uint32), "object_id": _touched(cap, np.uint32),
            "prev_index": _touched(cap, np.int32, -1)}


def _pool_ptrs(pool):
    return [_p(pool[k]) for k in ("position", "normal", "material_id", "object_id", "prev_index")]


def build_ppfl(scene, cfg, strategy=None, capacity=None, overalloc=10.0):
    """build_ppfl (fhv/storage.py:553-571)."""
    strategy = strategy or CaptureStrategy.one_view()
    assert strategy.kind == "one_view"
    w, h = cfg.resolution
    cap = int(w * h * overalloc) if capacity is None else int(capacity)
    plan, proj = _plan_args(scene, strategy, cfg)
    P, N, F, M, O = _tris(scene)
    pool = _new_pool(cap)
    heads = np.full(w * h, -1, np.int32)
    nf = np.zeros(1, np.int64)
    raw = np.zeros(4, np.int64)
    rc = lib().orc_build_ppfl(_i64(len(P)), _p(P), _p(N), _p(F), _p(M), _p(O), plan.res, _p(proj),
                              _i64(w), _i64(cap), *_pool_ptrs(pool), _p(heads), _p(nf), _p(raw))
    if rc not in (OK, OVERFLOW):
        raise OracleError(rc, "build_ppfl")
    return {"layout": "PPFL", "pool": pool, "heads": heads, "next_free": int(nf[0]),
            "capacity": cap, "overflowed": rc == OVERFLOW, "stats": _stats(plan, raw),
            "capture_resolution": h, "width": w, "height": h}


def build_pofl(scene, strategy, cfg, levels, capacity=None, overalloc=10.0):
    """build_pofl (fhv/storage.py:574-587)."""
    w, h = cfg.resolution
    cap = int(w * h * overalloc) if capacity is None else int(capacity)
    plan, proj = _plan_args(scene, strategy, cfg)
    P, N, F, M, O = _tris(scene)
    pool = _new_pool(cap)
    heads = np.full(8 ** levels, -1, np.int32)
    pyr = np.zeros(sum(8 ** k for k in range(levels)), np.uint8)
    nf = np.zeros(1, np.int64)
    raw = np.zeros(4, np.int64)
    rc = lib().orc_build_pofl(_i64(len(P)), _p(P), _p(N), _p(F), _p(M), _p(O), plan.strategy, plan.res,
                              _f64(plan.pitch), _p(proj), 3, levels, _i64(cap), *_pool_ptrs(pool),
                              _p(heads), _p(pyr), _p(nf), _p(raw))
    if rc not in (OK, OVERFLOW):
        raise OracleError(rc, "build_pofl")
    return {"layout": "POFL", "pool": pool, "heads": heads, "pyramid": pyr, "levels": levels,
            "next_free": int(nf[0]), "capacity": cap, "overflowed": rc == OVERFLOW,
            "stats": _stats(plan, raw), "capture_resolution": h}


def pofa_build(scene, strategy, cfg, levels):
    """pofa_build: count pass, exclusive scan, scatter pass (fhv/storage.py:590-621)."""
    plan, proj = _plan_args(scene, strategy, cfg)
    P, N, F, M, O = _tris(scene)
    c64 = _touched(8 ** levels, np.int64)
    raw1 = np.zeros(4, np.int64)
    rc = lib().orc_pofa_count(_i64(len(P)), _p(P), _p(N), _p(F), _p(M), _p(O), plan.strategy, plan.res,
                              _f64(plan.pitch), _p(proj), 3, levels, _p(c64), _p(raw1))
    if rc:
        raise OracleError(rc, "pofa_count")
    counts = np.zeros(8 ** levels, np.uint32)
    offsets = np.zeros(8 ** levels, np.uint32)
    total = np.zeros(1, np.int64)
    rc = lib().orc_pofa_offsets(_p(c64), levels, _p(counts), _p(offsets), _p(total))
    if rc:
        raise OracleError(rc, "pofa_offsets")
    n = int(total[0])
    pool = _new_pool(n)
    pyr = np.zeros(sum(8 ** k for k in range(levels)), np.uint8)
    raw2 = np.zeros(4, np.int64)
    rc = lib().orc_pofa_write(_i64(len(P)), _p(P), _p(N), _p(F), _p(M), _p(O), plan.strategy, plan.res,
                              _f64(plan.pitch), _p(proj), 3, levels, _p(offsets), _p(counts),
                              _i64(raw1[0]), *_pool_ptrs(pool), _p(pyr), _p(raw2))
    if rc:
        raise OracleError(rc, "pofa_write")
    return {"layout": "POFA", "pool": pool, "offsets": offsets, "counts": counts, "pyramid": pyr,
            "levels": levels, "next_free": n, "capacity": n, "overflowed": False,
            "stats": _stats(plan, raw2), "capture_resolution": int(cfg.resolution[1])}


def pyramid_from_occupancy(occ, levels):
    occ = np.ascontiguousarray(np.asarray(occ).astype(np.uint8))
    pyr = np.zeros(sum(8 ** k for k in range(levels)), np.uint8)
    lib().orc_pyramid_from_occupancy(_p(occ), levels, _p(pyr))
    return pyr


def cell_codes(pos32, levels):
    pos32 = np.ascontiguousarray(pos32, dtype=np.float32)
    out = np.zeros(len(pos32), np.int64)
    rc = lib().orc_cell_codes(_i64(len(pos32)), _p(pos32), levels, _p(out))
    if rc:
        raise OracleError(rc, "cell_codes")
    return out


def face_normals(positions):
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    out = np.zeros((len(pos), 3))
    lib().orc_face_normals(_i64(len(pos)), _p(pos), _p(out))
    return out


def splat(pool, n, camera, lights, radius, materials, background=(0.0, 0.0, 0.0, 0.0)):
    """splat_render (fhv/render.py:249-320) -> (rgba f64[h,w,4], depth f64[h,w], winner i64[h,w])."""
    w, h = camera.resolution
    cam = np.ascontiguousarray(camera.scalars())
    lk, lv, lc, la = pack_lights(lights)
    md, ms, msh, ma = pack_materials(materials)
    rgba = np.zeros((h, w, 4))
    depth = np.zeros((h, w))
    win = np.zeros((h, w), np.int64)
    pos = np.ascontiguousarray(pool["position"][:n])
    nrm = np.ascontiguousarray(pool["normal"][:n])
    mat = np.ascontiguousarray(pool["material_id"][:n])
    obj = np.ascontiguousarray(pool["object_id"][:n])
    bg = np.asarray(background, dtype=np.float64)
    rc = lib().orc_splat(_i64(n), _p(pos), _p(nrm), _p(mat), _p(obj), _p(cam), _f64(radius), _p(bg),
                         len(lights), _p(lk), _p(lv), _p(lc), _p(la), _p(md), _p(ms), _p(msh), _p(ma),
                         _p(rgba), _p(depth), _p(win))
    if rc:
        raise OracleError(rc, "splat")
    return rgba, depth, win


def primary_rays(camera):
    w, h = camera.resolution
    cam = np.ascontiguousarray(camera.scalars())
    o = np.zeros((w * h, 3))
    d = np.zeros((w * h, 3))
    lib().orc_primary_rays(_p(cam), _p(o), _p(d))
    return o, d


MODES = ("opaque_nearest", "transparency", "transparency_shadows")


def raycast(vol, camera, lights, radius, mode="transparency", cutoff=1.0, shadow_eps=None,
            materials=None, background=(0.0, 0.0, 0.0, 0.0), collect_ids=False, rows=None):
    """render_raycast compiled path (fhv/raycast.py:469-577) on an oracle volume
    dict.  Returns (rgba f64[h,w,4], stats dict, ids i32[h,w] or None).
    ``rows=(r0, r1)`` restricts the work to a row band (bench sampling)."""
    w, h = camera.resolution
    L = vol["levels"]
    o, d = primary_rays(camera)
    if vol["layout"] == "POFL":
        layout, a = 1, vol["heads"].astype(np.int64)
        b = vol["pool"]["prev_index"].astype(np.int64)
    else:
        layout, a, b = 0, vol["offsets"].astype(np.int64), vol["counts"].astype(np.int64)
    pyr_off = np.array([sum(8 ** j for j in range(k)) for k in range(L)], np.int64)
    lk, lv, lc, la = pack_lights(lights)
    md, ms, msh, ma = pack_materials(materials)
    eps = 2.0 * radius if shadow_eps is None else shadow_eps
    rgba = np.zeros((h * w, 4))
    bg = np.asarray(background, dtype=np.float64)
    rgba[:] = bg
    ids = np.full(h * w, -1, np.int32) if collect_ids else None
    counters = np.zeros(4, np.int64)
    pool = vol["pool"]
    r0, r1 = (0, h) if rows is None else rows
    cut = -1.0 if cutoff is None else float(cutoff)
    rc = lib().orc_raycast(_i64(r0 * w), _i64(r1 * w), _p(o), _p(d), layout, L, _p(a), _p(b),
                           _p(vol["pyramid"]), _p(pyr_off), _p(pool["position"]), _p(pool["normal"]),
                           _p(pool["material_id"]), _p(pool["object_id"]), _p(md), _p(ms), _p(msh),
                           _p(ma), len(lights), _p(lk), _p(lv), _p(lc), _p(la),
                           _p(np.ascontiguousarray(camera.eye)), _p(bg), _f64(radius), _f64(cut),
                           MODES.index(mode), _f64(eps), _p(rgba), _p(ids), _p(counters))
    if rc:
        raise OracleError(rc, "raycast")
    stats = dict(zip(("visited_leaves", "tested_fragments", "hits", "early_terminations"),
                     (int(c) for c in counters)))
    return rgba.reshape(h, w, 4), stats, (None if ids is None else ids.reshape(h, w))


def deferred(scene, camera, lights, background=(0.0, 0.0, 0.0, 0.0)):
    """deferred_baseline (fhv/render.py:327-382) -> dict of rgba f64[h,w,4],
    depth f64[h,w], G-buffer gpos/gnrm f64[h,w,3], gmat/gobj i32[h,w],
    valid bool[h,w], and the fragment count."""
    from paper_2211_15460_b200.raster import RasterConfig
    w, h = camera.resolution
    M = np.ascontiguousarray(RasterConfig.from_camera(camera).projection, dtype=np.float64)
    pos, vn, fn, mat, obj = _tris(scene)
    lk, lv, lc, la = pack_lights(lights)
    md, ms, msh, ma = pack_materials(scene.materials)
    out = {"rgba": np.zeros((h, w, 4)), "depth": np.zeros((h, w)), "gpos": np.zeros((h, w, 3)),
           "gnrm": np.zeros((h, w, 3)), "gmat": np.zeros((h, w), np.int32), "gobj": np.zeros((h, w), np.int32),
           "valid": np.zeros((h, w), np.uint8)}
    eye = np.ascontiguousarray(camera.eye, dtype=np.float64)
    bg = np.asarray(background, dtype=np.float64)
    n = ctypes.c_int64(0)
    rc = lib().orc_deferred(_i64(scene.n_triangles), _p(pos), _p(vn), _p(fn), _p(mat), _p(obj), _p(M), _i64(w),
                            _i64(h), _p(eye), len(lights), _p(lk), _p(lv), _p(lc), _p(la), _p(md), _p(ms), _p(msh),
                            _p(ma), _p(bg), _p(out["rgba"]), _p(out["depth"]), _p(out["gpos"]), _p(out["gnrm"]),
                            _p(out["gmat"]), _p(out["gobj"]), _p(out["valid"]), ctypes.byref(n))
    if rc:
        raise OracleError(rc, "deferred")
    out["valid"] = out["valid"].astype(bool)
    out["emitted"] = int(n.value)
    return out


_SNAP_HEADER = "<4s4sIIIIQ"  # magic, layout, levels, w, h, record size, count (fhv/storage.py:722-723)


def snapshot_bytes(vol):
    """FHV1 snapshot of an oracle volume dict (fhv/storage.py:725-755): header,
    directory, pyramid levels, packed 36-byte records of the stored prefix."""
    import struct
    from paper_2211_15460_b200.storage import RECORD_DTYPE
    n = min(vol["next_free"], vol["capacity"])
    if vol["layout"] == "PPFL":
        parts = [struct.pack(_SNAP_HEADER, b"FHV1", b"PPFL", 0, vol["width"], vol["height"], 36, n),
                 vol["heads"].astype("<i4").tobytes()]
    else:
        r = vol["capture_resolution"]
        parts = [struct.pack(_SNAP_HEADER, b"FHV1", vol["layout"].encode(), vol["levels"], r, r, 36, n)]
        if vol["layout"] == "POFL":
            parts.append(vol["heads"].astype("<i4").tobytes())
        else:
            parts += [vol["offsets"].astype("<u4").tobytes(), vol["counts"].astype("<u4").tobytes()]
        parts.append(vol["pyramid"].tobytes())
    rec = np.empty(n, dtype=RECORD_DTYPE)
    for k in RECORD_DTYPE.names:
        rec[k] = vol["pool"][k][:n]
    parts.append(rec.tobytes())
    return b"".join(parts)


def rebuild_pofl_as_pofa(vol):
    """rebuild_pofl_as_pofa (fhv/storage.py:624-652) of an oracle POFL dict:
    leaf codes of the f32 positions (cell_code), stable counting sort by leaf
    (emission = pool order inside a leaf), directory, pyramid; prev = -1."""
    L = vol["levels"]
    n = min(vol["next_free"], vol["capacity"])
    codes = cell_codes(vol["pool"]["position"][:n], L)
    counts = np.bincount(codes, minlength=8 ** L).astype(np.uint32)
    offsets = np.zeros(8 ** L, np.uint32)
    offsets[1:] = np.cumsum(counts[:-1], dtype=np.int64).astype(np.uint32)
    perm = np.argsort(codes, kind="stable")
    pool = _new_pool(n)
    for k in ("position", "normal", "material_id", "object_id"):
        pool[k][:] = vol["pool"][k][:n][perm]
    return {"layout": "POFA", "pool": pool, "offsets": offsets, "counts": counts,
            "pyramid": pyramid_from_occupancy(counts > 0, L), "levels": L, "next_free": n, "capacity": n,
            "overflowed": False, "capture_resolution": vol["capture_resolution"]}


# ---------------------------------------------------------------------------
# the reference's operator module, restated as plain Python loops (small
# cases only; checked against tests/golden/scalar.npz)


def coverage(ax, ay, bx, by, cx, cy, w, h):
    """coverage (fhv/_ckern.pyx:25-105 == fhv/_kernels_py.py:17-66): covered
    pixel centres in row-major order with barycentrics f_i / area2."""
    import math
    area2 = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax)
    if area2 <= 0.0:
        raise ValueError("coverage() requires positively wound vertices")
    x0 = max(0, math.ceil(min(ax, bx, cx) - 0.5))
    x1 = min(w - 1, math.floor(max(ax, bx, cx) - 0.5))
    y0 = max(0, math.ceil(min(ay, by, cy) - 0.5))
    y1 = min(h - 1, math.floor(max(ay, by, cy) - 0.5))
    d0x, d0y, d1x, d1y, d2x, d2y = cx - bx, cy - by, ax - cx, ay - cy, bx - ax, by - ay
    tl = [d0y < 0.0 or (d0y == 0.0 and d0x > 0.0), d1y < 0.0 or (d1y == 0.0 and d1x > 0.0),
          d2y < 0.0 or (d2y == 0.0 and d2x > 0.0)]
    px, py, lam = [], [], []
    for y in range(y0, y1 + 1):
        sy = y + 0.5
        for x in range(x0, x1 + 1):
            sx = x + 0.5
            f = (d0x * (sy - by) - d0y * (sx - bx), d1x * (sy - cy) - d1y * (sx - cx),
                 d2x * (sy - ay) - d2y * (sx - ax))
            if all(fi > 0.0 or (fi == 0.0 and t) for fi, t in zip(f, tl)):
                px.append(x)
                py.append(y)
                lam.append([fi / area2 for fi in f])
    return (np.array(px, np.int32), np.array(py, np.int32), np.array(lam, np.float64).reshape(-1, 3))


def linked_insert(keys, heads, prev, start) -> None:
    """linked_insert (fhv/_ckern.pyx:112-123), in place."""
    idx = int(start)
    for k in np.asarray(keys).tolist():
        prev[idx] = heads[k]
        heads[k] = idx
        idx += 1


def pofa_scatter(codes, offsets, counts, cursors, dest) -> int:
    """pofa_scatter (fhv/_ckern.pyx:126-143), in place; -1 or the first bad index."""
    for i, c in enumerate(np.asarray(codes).tolist()):
        cur = int(cursors[c])
        if cur >= int(counts[c]):
            return i
        dest[i] = int(offsets[c]) + cur
        cursors[c] = cur + 1
    return -1


def set_paths(pyramid_levels, codes, L) -> None:
    """OccupancyPyramid.set_paths (fhv/storage.py:294-301) on a list of level arrays."""
    for code in np.asarray(codes).tolist():
        for k in range(L):
            node = code >> (3 * (L - k))
            child = (code >> (3 * (L - k - 1))) & 7
            pyramid_levels[k][node] |= np.uint8(1 << child)
