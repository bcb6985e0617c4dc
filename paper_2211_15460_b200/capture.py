"""Raw fragment streams and the reference's sink-based capture_pass.

``capture_fragments`` runs the device rasteriser in list mode: every
fragment in the reference's emission order (job, y, x) with its f64 world
position/normal -- the ListSink view of capture (fhv/raster.py:309-320).
``capture_pass`` keeps the reference signature (fhv/raster.py:350-388): the
GPU produces all fragments, then the host hands them to ``sink`` one
FragmentBatch per job, in order.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .device import capture_cfg, device_scene
from .raster import CaptureStats, CaptureStrategy, FragmentBatch, RasterConfig, capture_plan

__all__ = ["capture_fragments", "capture_pass"]


def capture_fragments(scene, strategy: CaptureStrategy, cfg: RasterConfig, max_out: int | None = None,
                      device=None, depth: bool = False) -> dict:
    """``depth=True`` adds FragmentBatch.depth per fragment (screen
    strategies: lam @ ndc_z, fhv/raster.py:204; normal_space: 0.5)."""
    plan = capture_plan(scene, strategy, cfg)
    ds = device_scene(scene, device)
    dev = ds.device
    lib = _lib.load()
    cx, st = _lib.ctx(dev), _lib.stream_ptr(dev)
    tris, c = ds.struct(), capture_cfg(plan)
    n = _lib.c_i64(0)
    if max_out is None:
        rc = lib.fhv_capture_list(cx, tris, c, 0, None, None, None, None, None, n, st)
        _lib.check(rc, "capture_fragments")
        max_out = int(n.value)
    job = torch.empty(max_out, dtype=torch.int64, device=dev)
    px = torch.empty(max_out, dtype=torch.int32, device=dev)
    py = torch.empty(max_out, dtype=torch.int32, device=dev)
    wpos = torch.empty((max_out, 3), dtype=torch.float64, device=dev)
    wnrm = torch.empty((max_out, 3), dtype=torch.float64, device=dev)
    dep = torch.empty(max_out, dtype=torch.float64, device=dev) if depth else None
    rc = lib.fhv_capture_list_depth(cx, tris, c, max_out, _lib.ptr(job), _lib.ptr(px), _lib.ptr(py), _lib.ptr(wpos),
                                    _lib.ptr(wnrm), _lib.ptr(dep), n, st)
    _lib.check(rc, "capture_fragments")
    total = int(n.value)
    k = min(total, max_out)
    out = {"job": job[:k], "raster_x": px[:k], "raster_y": py[:k], "world_position": wpos[:k],
           "world_normal": wnrm[:k], "stats": plan.stats(total), "plan": plan}
    if depth:
        out["depth"] = dep[:k]
    return out


def capture_pass(scene, strategy: CaptureStrategy, cfg: RasterConfig, sink, threads: int = 1,
                 device=None) -> CaptureStats:
    """Reference-compatible capture_pass: device rasterisation, host sink calls."""
    out = capture_fragments(scene, strategy, cfg, device=device, depth=True)
    plan = out["plan"]
    job = out["job"].cpu().numpy()
    if len(job):
        px = out["raster_x"].cpu().numpy()
        py = out["raster_y"].cpu().numpy()
        wp = out["world_position"].cpu().numpy()
        wn = out["world_normal"].cpu().numpy()
        dp = out["depth"].cpu().numpy()
        cuts = np.flatnonzero(np.diff(job)) + 1
        starts = np.concatenate(([0], cuts))
        ends = np.concatenate((cuts, [len(job)]))
        T = scene.n_triangles
        for s, e in zip(starts, ends):
            j = int(job[s])
            t = j % T if plan.strategy == 1 else (j // 3 if plan.strategy == 2 else j)
            sink(FragmentBatch(px[s:e], py[s:e], wp[s:e], wn[s:e], dp[s:e], int(scene.material_id[t]),
                               int(scene.object_id[t])))
    return out["stats"]
