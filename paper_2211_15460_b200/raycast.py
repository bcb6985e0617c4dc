"""Octree ray casting on the device (render_raycast, fhv/raycast.py:469-577).

Primary rays are generated inside the kernel with primary_rays' exact
elementwise arithmetic; traversal, per-leaf hit sorting, compositing,
early termination, shadow rays and RaycastStats run in
``csrc/fhv_raycast.cu``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import DeviceShading, host_f64
from .lights import ImageBuffer
from .scene import Camera, Material, SceneError

__all__ = ["RAYCAST_MODES", "RaycastConfig", "RaycastStats", "default_raycast_config", "primary_rays",
           "render_raycast", "render_raycast_rays"]

RAYCAST_MODES = ("opaque_nearest", "transparency", "transparency_shadows")


@dataclass(frozen=True)
class RaycastConfig:
    """Splat radius, termination threshold, mode, shadow offset (fhv/raycast.py:68-86)."""

    splat_radius_world: float
    alpha_cutoff: float | None = 1.0
    mode: str = "transparency"
    shadow_epsilon: float = 1e-3

    def __post_init__(self):
        if self.splat_radius_world <= 0.0:
            raise SceneError("splat radius must be > 0")
        if self.alpha_cutoff is not None and not 0.0 < self.alpha_cutoff <= 1.0:
            raise SceneError("alpha_cutoff must be in (0,1] or None")
        if self.mode not in RAYCAST_MODES:
            raise SceneError(f"unknown raycast mode {self.mode!r}")


def default_raycast_config(fhv, mode: str = "transparency", alpha_cutoff: float | None = 1.0,
                           splat_radius: float | None = None, shadow_epsilon: float | None = None) -> RaycastConfig:
    """radius = min(footprint/sqrt(2), half a leaf edge); eps = 2r (fhv/raycast.py:89-100)."""
    footprint = 1.0 / fhv.capture_resolution
    cap = 0.5 / (1 << fhv.levels)
    r = footprint / math.sqrt(2.0) if splat_radius is None else splat_radius
    r = min(r, cap) if splat_radius is None else r
    eps = 2.0 * r if shadow_epsilon is None else shadow_epsilon
    return RaycastConfig(r, alpha_cutoff, mode, eps)


@dataclass
class RaycastStats:
    visited_leaves: int = 0
    tested_fragments: int = 0
    hits: int = 0
    early_terminations: int = 0

    def merge(self, other: "RaycastStats") -> None:
        self.visited_leaves += other.visited_leaves
        self.tested_fragments += other.tested_fragments
        self.hits += other.hits
        self.early_terminations += other.early_terminations

    def as_dict(self) -> dict:
        return {"visited_leaves": self.visited_leaves, "tested_fragments": self.tested_fragments,
                "hits": self.hits, "early_terminations": self.early_terminations}


def primary_rays(camera: Camera):
    """(origins, directions) per pixel, row-major, NumPy host arrays -- the
    reference helper (fhv/raycast.py:148-172); the device kernel recomputes
    the same values itself."""
    w, h = camera.resolution
    rr, uu, ff = camera.basis()
    xs = (np.arange(w, dtype=np.float64) + 0.5) / w * 2.0 - 1.0
    ys = 1.0 - (np.arange(h, dtype=np.float64) + 0.5) / h * 2.0
    nx = np.broadcast_to(xs[None, :], (h, w)).ravel()
    ny = np.broadcast_to(ys[:, None], (h, w)).ravel()
    if camera.kind == "orthographic":
        hh = camera.extent_or_fov / 2.0
        hw = hh * camera.aspect
        o = camera.eye[None, :] + nx[:, None] * (hw * rr)[None, :] + ny[:, None] * (hh * uu)[None, :] \
            + (camera.near * ff)[None, :]
        return o, np.broadcast_to(ff, o.shape).copy()
    t = math.tan(math.radians(camera.extent_or_fov) / 2.0)
    d = ff[None, :] + nx[:, None] * (t * camera.aspect * rr)[None, :] + ny[:, None] * (t * uu)[None, :]
    d = d / np.linalg.norm(d, axis=1, keepdims=True)
    return np.broadcast_to(camera.eye, d.shape).copy(), d


def _volume(fhv) -> "_lib.Volume":
    pool = fhv.pool
    if fhv.layout == "POFA":
        return _lib.Volume(0, fhv.levels, _lib.ptr(fhv.directory.offsets), _lib.ptr(fhv.directory.counts), None, None,
                           _lib.ptr(fhv.pyramid.data), _lib.ptr(pool.position), _lib.ptr(pool.normal),
                           _lib.ptr(pool.material_id), _lib.ptr(pool.object_id))
    if fhv.layout == "POFL":
        return _lib.Volume(1, fhv.levels, None, None, _lib.ptr(fhv.directory.heads), _lib.ptr(pool.prev_index),
                           _lib.ptr(fhv.pyramid.data), _lib.ptr(pool.position), _lib.ptr(pool.normal),
                           _lib.ptr(pool.material_id), _lib.ptr(pool.object_id))
    raise SceneError("ray casting requires a per-octant layout")


def render_raycast(fhv, camera: Camera, lights, cfg: RaycastConfig | None = None, materials=None,
                   background=(0.0, 0.0, 0.0, 0.0), threads: int = 1, collect_ids: bool = False, *,
                   rows: tuple | None = None, out: ImageBuffer | None = None, sync: bool = True,
                   shading: DeviceShading | None = None):
    """Ray-cast every pixel; returns (ImageBuffer, RaycastStats[, ids]) with
    CUDA tensors.  ``threads`` is accepted and ignored.  ``rows=(r0, r1)``
    renders a row band only (multi-GPU slabs)."""
    if fhv.layout not in ("POFA", "POFL"):
        raise SceneError("ray casting requires a per-octant layout")
    if cfg is None:
        cfg = default_raycast_config(fhv)
    if materials is None:
        materials = fhv.materials or [Material()]
    dev = fhv.pool.device
    w, h = camera.resolution
    if out is None:
        px = torch.empty((h, w, 4), dtype=torch.float64, device=dev)
        px[:] = torch.tensor(background, dtype=torch.float64, device=dev)
        out = ImageBuffer(w, h, px, torch.full((h, w), float("inf"), dtype=torch.float64, device=dev))
    ids = torch.full((h, w), -1, dtype=torch.int32, device=dev) if collect_ids else None
    counters = torch.zeros(4, dtype=torch.int64, device=dev)
    if shading is None:
        shading = DeviceShading(materials, lights, dev)
    cam = host_f64(camera.scalars())
    bg = host_f64(background)
    r0, r1 = (0, h) if rows is None else rows
    cutoff = -1.0 if cfg.alpha_cutoff is None else float(cfg.alpha_cutoff)
    lib = _lib.load()
    rc = lib.fhv_raycast(_lib.ctx(dev), _volume(fhv), shading.struct(), cam.ctypes.data, bg.ctypes.data,
                         float(cfg.splat_radius_world), cutoff, RAYCAST_MODES.index(cfg.mode),
                         float(cfg.shadow_epsilon), r0, r1, _lib.ptr(out.pixels), _lib.ptr(ids), _lib.ptr(counters),
                         _lib.stream_ptr(dev))
    _lib.check(rc, "render_raycast")
    stats = RaycastStats()
    if sync:
        c = counters.cpu().tolist()
        stats = RaycastStats(*c)
    else:
        stats.counters = counters  # type: ignore[attr-defined]
    if collect_ids:
        return out, stats, ids
    return out, stats


def render_raycast_rays(fhv, origins: torch.Tensor, dirs: torch.Tensor, eye, lights, cfg: RaycastConfig,
                        materials=None, background=(0.0, 0.0, 0.0, 0.0), start: int = 0, end: int | None = None,
                        out_rgba: torch.Tensor | None = None, ids: torch.Tensor | None = None):
    """raycast_image 1:1 (fhv/_ckern.pyx:653-743): caller-provided rays."""
    dev = fhv.pool.device
    P = origins.shape[0]
    end = P if end is None else end
    if out_rgba is None:
        out_rgba = torch.empty((P, 4), dtype=torch.float64, device=dev)
        out_rgba[:] = torch.tensor(background, dtype=torch.float64, device=dev)
    counters = torch.zeros(4, dtype=torch.int64, device=dev)
    shading = DeviceShading(materials or fhv.materials or [Material()], lights, dev)
    cutoff = -1.0 if cfg.alpha_cutoff is None else float(cfg.alpha_cutoff)
    e, bg = host_f64(eye), host_f64(background)
    lib = _lib.load()
    rc = lib.fhv_raycast_image(_lib.ctx(dev), start, end, _lib.ptr(origins.contiguous()), _lib.ptr(dirs.contiguous()),
                               _volume(fhv), shading.struct(), e.ctypes.data, bg.ctypes.data,
                               float(cfg.splat_radius_world), cutoff, RAYCAST_MODES.index(cfg.mode),
                               float(cfg.shadow_epsilon), _lib.ptr(out_rgba), _lib.ptr(ids), _lib.ptr(counters),
                               _lib.stream_ptr(dev))
    _lib.check(rc, "raycast_image")
    return out_rgba, RaycastStats(*counters.cpu().tolist())
