"""The reference's operator module on the device: ``fhv._backend.kernels()``
(fhv/_backend.py:25-29) returns a module with ``BACKEND_NAME`` and
``coverage`` / ``linked_insert`` / ``pofa_scatter`` / ``raycast_image``
(fhv/_ckern.pyx:25-143, 653-743).  This module has the same four calls with
the same argument meaning, return values and in-place mutation, executed by
the CUDA kernels behind ``include/fhv_b200.h`` (``fhv_op_coverage``,
``fhv_op_linked_insert``, ``fhv_op_pofa_scatter``, ``fhv_raycast_image``).

Arguments may be NumPy arrays (the reference's types: results come back into
them in place) or CUDA tensors (mutated on the device).  The capture drivers
of this package never call these per triangle -- the fused capture kernels do
the same work per fragment; ``coverage_batch`` is the batched form.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .device import default_device

BACKEND_NAME = "b200"

__all__ = ["BACKEND_NAME", "coverage", "coverage_batch", "linked_insert", "pofa_scatter", "raycast_image"]


def _dev_of(*arrays):
    for a in arrays:
        if isinstance(a, torch.Tensor) and a.is_cuda:
            return a.device
    return default_device()


def _to_dev(a, dtype: torch.dtype, dev) -> torch.Tensor:
    """Device copy (or view) of ``a`` with ``dtype``, contiguous."""
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dtype)


def _write_back(dst, src: torch.Tensor) -> None:
    """Copy a device result into the caller's array (in place)."""
    if isinstance(dst, torch.Tensor):
        if dst.data_ptr() != src.data_ptr():
            dst.copy_(src.to(dst.dtype).reshape(dst.shape))
        return
    h = src.cpu().numpy()
    dst[...] = h.reshape(dst.shape).astype(dst.dtype, copy=False)


def coverage_batch(v6, wh, device=None, max_out: int | None = None) -> dict:
    """coverage() of n triangles in one launch pair: v6 (n, 6) f64
    (ax, ay, bx, by, cx, cy), wh (n, 2) int32.  Returns device tensors
    ``tri_off`` (n+1), ``px``, ``py``, ``l0``, ``l1``, ``l2`` (triangle-major,
    row-major inside each), and ``first_bad`` (first triangle with
    area2 <= 0, or -1)."""
    dev = default_device(device) if device is not None else _dev_of(v6, wh)
    tv = _to_dev(v6, torch.float64, dev).reshape(-1, 6)
    tw = _to_dev(wh, torch.int32, dev).reshape(-1, 2)
    n = tv.shape[0]
    if tw.shape[0] != n:
        raise ValueError("coverage_batch: v6 and wh disagree in length")
    lib = _lib.load()
    cx, st = _lib.ctx(dev), _lib.stream_ptr(dev)
    off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    total, bad = ctypes.c_int64(0), ctypes.c_int64(-1)
    if max_out is None:
        rc = lib.fhv_op_coverage(cx, n, _lib.ptr(tv), _lib.ptr(tw), 0, _lib.ptr(off), None, None, None, None, None,
                                 ctypes.byref(total), ctypes.byref(bad), st)
        _lib.check(rc, "coverage")
        max_out = int(total.value)
    px = torch.empty(max_out, dtype=torch.int32, device=dev)
    py = torch.empty(max_out, dtype=torch.int32, device=dev)
    l0, l1, l2 = (torch.empty(max_out, dtype=torch.float64, device=dev) for _ in range(3))
    rc = lib.fhv_op_coverage(cx, n, _lib.ptr(tv), _lib.ptr(tw), max_out, _lib.ptr(off), _lib.ptr(px), _lib.ptr(py),
                             _lib.ptr(l0), _lib.ptr(l1), _lib.ptr(l2), ctypes.byref(total), ctypes.byref(bad), st)
    _lib.check(rc, "coverage")
    k = min(int(total.value), max_out)
    return {"tri_off": off, "px": px[:k], "py": py[:k], "l0": l0[:k], "l1": l1[:k], "l2": l2[:k],
            "total": int(total.value), "first_bad": int(bad.value)}


def coverage(ax, ay, bx, by, cx, cy, w, h):
    """Pixel-centre coverage of one raster-space triangle (fhv/_ckern.pyx:25-105):
    ``(px, py, l0, l1, l2)`` NumPy arrays (int32, int32, f64 x 3), row-major.
    Raises ValueError unless the doubled signed area is positive."""
    v = np.array([[ax, ay, bx, by, cx, cy]], dtype=np.float64)
    r = coverage_batch(v, np.array([[w, h]], dtype=np.int32))
    if r["first_bad"] >= 0:
        raise ValueError("coverage() requires positively wound vertices")
    return (r["px"].cpu().numpy(), r["py"].cpu().numpy(), r["l0"].cpu().numpy(), r["l1"].cpu().numpy(),
            r["l2"].cpu().numpy())


def linked_insert(keys, heads, prev, start) -> None:
    """Chain ``len(keys)`` records from pool index ``start`` (fhv/_ckern.pyx:112-123):
    ``prev[start+i] = heads[keys[i]]; heads[keys[i]] = start+i`` in order.
    ``heads`` / ``prev`` (int32) are updated in place."""
    dev = _dev_of(keys, heads, prev)
    tk = _to_dev(keys, torch.int64, dev).reshape(-1)
    th = heads if isinstance(heads, torch.Tensor) and heads.is_cuda and heads.dtype == torch.int32 \
        and heads.is_contiguous() else _to_dev(heads, torch.int32, dev)
    tp = prev if isinstance(prev, torch.Tensor) and prev.is_cuda and prev.dtype == torch.int32 \
        and prev.is_contiguous() else _to_dev(prev, torch.int32, dev)
    n = tk.numel()
    if n == 0:
        return
    start = int(start)
    if start < 0 or start + n > tp.numel():
        raise IndexError(f"linked_insert: records [{start}, {start + n}) outside prev of length {tp.numel()}")
    rc = _lib.load().fhv_op_linked_insert(_lib.ctx(dev), n, _lib.ptr(tk), th.numel(), _lib.ptr(th), _lib.ptr(tp),
                                          tp.numel(), start, _lib.stream_ptr(dev))
    if rc == _lib.FHV_BAD_ARGS:
        raise IndexError("linked_insert: key outside the directory")
    _lib.check(rc, "linked_insert")
    _write_back(heads, th)
    _write_back(prev, tp)


def pofa_scatter(codes, offsets, counts, cursors, dest) -> int:
    """``dest[i] = offsets[c] + cursors[c]++`` in order (fhv/_ckern.pyx:126-143).
    Returns -1, or the index of the first fragment whose leaf cursor would
    pass its count (nothing from it on is written).  ``cursors`` (uint32) and
    ``dest`` (int64) are updated in place."""
    dev = _dev_of(codes, offsets, counts, cursors, dest)
    tc = _to_dev(codes, torch.int64, dev).reshape(-1)
    n = tc.numel()
    if n == 0:
        return -1

    def u32(a):
        if isinstance(a, torch.Tensor) and a.is_cuda and a.dtype == torch.uint32 and a.is_contiguous():
            return a
        if isinstance(a, np.ndarray):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).to(dev).view(torch.uint32)
        return a.to(dev).contiguous().view(torch.int32).view(torch.uint32) if a.dtype in (torch.uint32, torch.int32) \
            else a.to(device=dev, dtype=torch.int64).to(torch.int32).view(torch.uint32)
    to, tn, tcur = u32(offsets), u32(counts), u32(cursors)
    td = dest if isinstance(dest, torch.Tensor) and dest.is_cuda and dest.dtype == torch.int64 \
        and dest.is_contiguous() else _to_dev(dest, torch.int64, dev)
    if td.numel() < n:
        raise IndexError("pofa_scatter: dest shorter than codes")
    bad = ctypes.c_int64(-1)
    rc = _lib.load().fhv_op_pofa_scatter(_lib.ctx(dev), n, _lib.ptr(tc), tn.numel(), _lib.ptr(to), _lib.ptr(tn),
                                         _lib.ptr(tcur), _lib.ptr(td), ctypes.byref(bad), _lib.stream_ptr(dev))
    if rc == _lib.FHV_BAD_ARGS:
        raise IndexError("pofa_scatter: code outside the directory")
    _lib.check(rc, "pofa_scatter")
    if isinstance(cursors, np.ndarray):
        cursors[...] = tcur.view(torch.int32).cpu().numpy().view(np.uint32).reshape(cursors.shape)
    elif cursors.data_ptr() != tcur.data_ptr():
        cursors.copy_(tcur.view(torch.int32).to(torch.int64).remainder(1 << 32).to(cursors.dtype))
    _write_back(dest, td)
    return int(bad.value)


def raycast_image(start_pix, end_pix, origins, dirs, layout_kind, levels, arr_a, arr_b, pyramid, pyr_off,
                  pool_pos, pool_nrm, pool_mat, pool_obj, mat_diffuse, mat_specular, mat_shininess, mat_alpha,
                  light_kind, light_vec, light_color, light_ambient, eye, background, radius, cutoff, mode,
                  shadow_eps, out_rgba, out_ids, counters) -> None:
    """Evaluate primary rays [start_pix, end_pix) (fhv/_ckern.pyx:653-743),
    same arguments: writes ``out_rgba`` rows and ``out_ids`` (when non-empty)
    in place, adds the four RaycastStats counters into ``counters``."""
    levels = int(levels)
    if levels < 1 or levels > 24:
        raise ValueError("levels out of range")
    if levels > 12:
        raise ValueError("levels > 12: the B200 ray caster keeps 8^L-leaf pyramids up to L = 12")
    dev = _dev_of(origins, dirs, arr_a, pool_pos, out_rgba)
    f64 = lambda a: _to_dev(a, torch.float64, dev)  # noqa: E731
    # the flattened pyramid: level k at pyr_off[k] (this layout: (8^k - 1) / 7)
    offs = [int(v) for v in np.asarray(pyr_off.cpu() if isinstance(pyr_off, torch.Tensor) else pyr_off)]
    tp = _to_dev(pyramid, torch.uint8, dev)
    std = [((1 << (3 * k)) - 1) // 7 for k in range(levels)]
    if offs[:levels] != std:
        tp = torch.cat([tp[offs[k]:offs[k] + (1 << (3 * k))] for k in range(levels)])
    if int(layout_kind) == 0:  # POFA: offsets, counts
        a = _to_dev(arr_a, torch.int64, dev).to(torch.int32).view(torch.uint32)
        b = _to_dev(arr_b, torch.int64, dev).to(torch.int32).view(torch.uint32)
        vol = (0, a, b, None, None)
    else:  # POFL: heads, prev
        a = _to_dev(arr_a, torch.int64, dev).to(torch.int32)
        b = _to_dev(arr_b, torch.int64, dev).to(torch.int32)
        vol = (1, None, None, a, b)
    pos = _to_dev(pool_pos, torch.float32, dev)
    nrm = _to_dev(pool_nrm, torch.float32, dev)
    mat = _to_dev(pool_mat, torch.int64, dev).to(torch.int32).view(torch.uint32)
    obj = _to_dev(pool_obj, torch.int64, dev).to(torch.int32).view(torch.uint32)
    v = _lib.Volume(vol[0], levels, _lib.ptr(vol[1]), _lib.ptr(vol[2]), _lib.ptr(vol[3]), _lib.ptr(vol[4]),
                    _lib.ptr(tp), _lib.ptr(pos), _lib.ptr(nrm), _lib.ptr(mat), _lib.ptr(obj))
    lk = _to_dev(light_kind, torch.uint8, dev)
    tabs = [lk, f64(light_vec), f64(light_color), f64(light_ambient), f64(mat_diffuse), f64(mat_specular),
            f64(mat_shininess), f64(mat_alpha)]
    sh = _lib.Shading(lk.numel(), *[_lib.ptr(t) for t in tabs[:4]], tabs[6].numel(), *[_lib.ptr(t) for t in tabs[4:]])
    to, td = f64(origins).reshape(-1, 3), f64(dirs).reshape(-1, 3)
    rgba = out_rgba if isinstance(out_rgba, torch.Tensor) and out_rgba.is_cuda and out_rgba.dtype == torch.float64 \
        and out_rgba.is_contiguous() else f64(out_rgba)
    has_ids = (out_ids.numel() if isinstance(out_ids, torch.Tensor) else np.asarray(out_ids).size) > 0
    ids = None
    if has_ids:
        ids = out_ids if isinstance(out_ids, torch.Tensor) and out_ids.is_cuda and out_ids.dtype == torch.int32 \
            and out_ids.is_contiguous() else _to_dev(out_ids, torch.int32, dev)
    cnt = torch.zeros(4, dtype=torch.int64, device=dev)
    e = np.ascontiguousarray(np.asarray(eye.cpu() if isinstance(eye, torch.Tensor) else eye, dtype=np.float64))
    bg = np.ascontiguousarray(np.asarray(background.cpu() if isinstance(background, torch.Tensor) else background,
                                         dtype=np.float64))
    rc = _lib.load().fhv_raycast_image(_lib.ctx(dev), int(start_pix), int(end_pix), _lib.ptr(to), _lib.ptr(td), v,
                                       sh, e.ctypes.data, bg.ctypes.data, float(radius), float(cutoff), int(mode),
                                       float(shadow_eps), _lib.ptr(rgba), _lib.ptr(ids), _lib.ptr(cnt),
                                       _lib.stream_ptr(dev))
    _lib.check(rc, "raycast_image")
    _write_back(out_rgba, rgba)
    if has_ids:
        _write_back(out_ids, ids)
    c = cnt.cpu()
    if isinstance(counters, torch.Tensor):
        counters += c.to(counters.device)
    else:
        counters += c.numpy()
