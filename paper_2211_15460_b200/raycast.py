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

__all__ = ["HitRecord", "RAYCAST_MODES", "Ray", "RaycastConfig", "RaycastStats", "default_raycast_config",
           "gather_ray_hits", "gen_primary_ray", "intersect_fragment", "primary_rays", "raycast_pixel",
           "render_raycast", "render_raycast_rays", "shadow_transmittance", "traverse_octree"]

RAYCAST_MODES = ("opaque_nearest", "transparency", "transparency_shadows")


@dataclass
class Ray:
    """A ray with its parameter interval (fhv/raycast.py:42-58); the direction
    is unit-normalised unless it is already within 1e-9 of unit length."""

    origin: np.ndarray
    direction: np.ndarray
    t_min: float = 0.0
    t_max: float = math.inf

    def __post_init__(self):
        self.origin = np.asarray(self.origin, dtype=np.float64)
        self.direction = np.asarray(self.direction, dtype=np.float64)
        n = float(np.linalg.norm(self.direction))
        if abs(n - 1.0) > 1e-9:
            if n == 0.0:
                raise SceneError("zero ray direction")
            self.direction = self.direction / n
        if not self.t_min < self.t_max:
            raise SceneError("ray needs t_min < t_max")


@dataclass
class HitRecord:
    t: float
    fragment_index: int
    leaf: int


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


# ---------------------------------------------------------------------------
# scalar queries (fhv/raycast.py:129-453) -- each one a small device launch
# over the resident volume (fhv_ray_probe / fhv_transmittance /
# fhv_leaf_order / fhv_intersect_points); hit lists come back to the host


def gen_primary_ray(camera: Camera, px) -> Ray:
    """Ray through the centre of pixel (ix, iy) (fhv/raycast.py:129-145)."""
    ix, iy = px
    w, h = camera.resolution
    if not (0 <= ix < w and 0 <= iy < h):
        raise SceneError(f"pixel {px} outside resolution")
    r, u, f = camera.basis()
    ndc_x = (ix + 0.5) / w * 2.0 - 1.0
    ndc_y = 1.0 - (iy + 0.5) / h * 2.0
    if camera.kind == "orthographic":
        half_h = camera.extent_or_fov / 2.0
        half_w = half_h * camera.aspect
        origin = camera.eye + ndc_x * half_w * r + ndc_y * half_h * u + camera.near * f
        return Ray(origin, f.copy())
    t = math.tan(math.radians(camera.extent_or_fov) / 2.0)
    direction = f + ndc_x * t * camera.aspect * r + ndc_y * t * u
    return Ray(camera.eye.copy(), direction)


def _dev_ray(ray: Ray, dev):
    o = torch.from_numpy(np.ascontiguousarray(ray.origin, dtype=np.float64)).to(dev)
    d = torch.from_numpy(np.ascontiguousarray(ray.direction, dtype=np.float64)).to(dev)
    return o, d


def _merge(stats: RaycastStats | None, c, hits: bool = True) -> None:
    if stats is None:
        return
    stats.visited_leaves += int(c[0])
    stats.tested_fragments += int(c[1])
    if hits:
        stats.hits += int(c[2])
        stats.early_terminations += int(c[3])


def traverse_octree(pyramid, ray: Ray, visit) -> int:
    """Visit the occupied leaves the ray crosses, nearest entry first
    (fhv/raycast.py:205-243): ``visit(code, t_enter, t_exit) -> bool``, False
    stops.  Returns the number of leaves visited.  The device lists the leaf
    sequence (it does not depend on the visitor); the host replays it."""
    dev = pyramid.data.device
    o, d = _dev_ray(ray, dev)
    lib = _lib.load()
    cap = 1024
    while True:
        codes = torch.empty(cap, dtype=torch.int64, device=dev)
        te = torch.empty(cap, dtype=torch.float64, device=dev)
        tx = torch.empty(cap, dtype=torch.float64, device=dev)
        n = torch.zeros(1, dtype=torch.int64, device=dev)
        rc = lib.fhv_leaf_order(_lib.ctx(dev), pyramid.leaf_levels, _lib.ptr(pyramid.data), _lib.ptr(o), _lib.ptr(d),
                                float(ray.t_min), float(ray.t_max), cap, _lib.ptr(codes), _lib.ptr(te), _lib.ptr(tx),
                                _lib.ptr(n), _lib.stream_ptr(dev))
        _lib.check(rc, "traverse_octree")
        total = int(n.item())
        if total <= cap:
            break
        cap = total
    visited = 0
    for code, a, b in zip(codes[:total].tolist(), te[:total].tolist(), tx[:total].tolist()):
        visited += 1
        if not visit(code, a, b):
            break
    return visited


def intersect_fragment(ray: Ray, position, radius: float, device=None) -> float | None:
    """Hit parameter of a point fragment within the splat radius, or None
    (fhv/raycast.py:246-262)."""
    from .device import default_device
    dev = default_device(device)
    p = torch.from_numpy(np.ascontiguousarray(np.asarray(position, dtype=np.float64).reshape(1, 3))).to(dev)
    t = torch.empty(1, dtype=torch.float64, device=dev)
    hit = torch.empty(1, dtype=torch.int8, device=dev)
    o, dr = host_f64(ray.origin), host_f64(ray.direction)
    rc = _lib.load().fhv_intersect_points(_lib.ctx(dev), 1, _lib.ptr(p), o.ctypes.data, dr.ctypes.data,
                                          float(ray.t_min), float(ray.t_max), float(radius), _lib.ptr(t),
                                          _lib.ptr(hit), _lib.stream_ptr(dev))
    _lib.check(rc, "intersect_fragment")
    return float(t.item()) if int(hit.item()) else None


def _probe(fhv, ray: Ray, mode: int, radius: float, shading: DeviceShading, cutoff: float, shadow_eps: float,
           background, eye):
    dev = fhv.pool.device
    o, d = _dev_ray(ray, dev)
    tmin = torch.tensor([float(ray.t_min)], dtype=torch.float64, device=dev)
    tmax = torch.tensor([float(ray.t_max)], dtype=torch.float64, device=dev)
    rgba = torch.empty(4, dtype=torch.float64, device=dev)
    hit_n = torch.zeros(1, dtype=torch.int64, device=dev)
    stats = torch.zeros(4, dtype=torch.int64, device=dev)
    bg = host_f64(background)
    e = None if eye is None else host_f64(eye)
    lib = _lib.load()
    cap = 256
    while True:
        ht = torch.empty(cap, dtype=torch.float64, device=dev)
        hi = torch.empty(cap, dtype=torch.int64, device=dev)
        hl = torch.empty(cap, dtype=torch.int64, device=dev)
        rc = lib.fhv_ray_probe(_lib.ctx(dev), 1, _lib.ptr(o), _lib.ptr(d), _lib.ptr(tmin), _lib.ptr(tmax),
                               _volume(fhv), shading.struct(), None if e is None else e.ctypes.data, bg.ctypes.data,
                               float(radius), float(cutoff), mode, float(shadow_eps), cap, _lib.ptr(rgba),
                               _lib.ptr(ht), _lib.ptr(hi), _lib.ptr(hl), _lib.ptr(hit_n), _lib.ptr(stats),
                               _lib.stream_ptr(dev))
        _lib.check(rc, "raycast_pixel")
        n = int(hit_n.item())
        if n <= cap:
            break
        cap = n
    hits = [HitRecord(t, i, c) for t, i, c in zip(ht[:n].tolist(), hi[:n].tolist(), hl[:n].tolist())]
    return rgba.cpu().numpy(), hits, stats.cpu().tolist()


def _shading_for(fhv, materials, lights, dev) -> DeviceShading:
    if materials is None:
        materials = fhv.materials or [Material()]
    if isinstance(materials, dict):
        return DeviceShading.from_arrays(materials, lights, dev)
    return DeviceShading(materials, lights, dev)


def gather_ray_hits(fhv, ray: Ray, radius: float, stats: RaycastStats | None = None) -> list:
    """Every hit along a ray, leaf by leaf, sorted by (t, index) inside each
    leaf (fhv/raycast.py:294-308)."""
    if fhv.layout not in ("POFA", "POFL"):
        raise SceneError("ray casting requires a per-octant layout")
    sh = _shading_for(fhv, None, [], fhv.pool.device)
    _, hits, c = _probe(fhv, ray, 3, radius, sh, -1.0, 0.0, (0.0, 0.0, 0.0, 0.0), None)
    _merge(stats, c, hits=False)
    return hits


def raycast_pixel(fhv, ray: Ray, lights, cfg: RaycastConfig, materials=None, background=(0.0, 0.0, 0.0, 0.0),
                  eye=None, stats: RaycastStats | None = None, hit_out: list | None = None) -> np.ndarray:
    """Evaluate one ray against a per-octant volume; returns rgba
    (fhv/raycast.py:351-405).  ``eye`` defaults to the ray origin; ``hit_out``
    receives the HitRecords composited (opaque_nearest: the first)."""
    if fhv.layout not in ("POFA", "POFL"):
        raise SceneError("ray casting requires a per-octant layout")
    sh = _shading_for(fhv, materials, lights, fhv.pool.device)
    cutoff = -1.0 if cfg.alpha_cutoff is None else float(cfg.alpha_cutoff)
    rgba, hits, c = _probe(fhv, ray, RAYCAST_MODES.index(cfg.mode), cfg.splat_radius_world, sh, cutoff,
                           cfg.shadow_epsilon, background, eye)
    _merge(stats, c)
    if hit_out is not None:
        hit_out.extend(hits)
    return rgba


def shadow_transmittance(fhv, point, light, cfg: RaycastConfig, exclude_object_id: int | None = None,
                         exclude_cell: int | None = None, stats: RaycastStats | None = None,
                         alpha_table=None) -> float:
    """Product of (1 - alpha) over the fragments between a point and a light
    (fhv/raycast.py:408-453); fragments of the excluded (object id, leaf)
    pair are skipped when both are given."""
    dev = fhv.pool.device
    if alpha_table is not None:
        a = np.asarray(alpha_table, dtype=np.float64).reshape(-1)
        z = np.zeros((len(a), 3))
        sh = DeviceShading.from_arrays({"diffuse": z, "specular": z, "shininess": np.zeros(len(a)), "alpha": a},
                                       [light], dev)
    else:
        sh = _shading_for(fhv, None, [light], dev)
    p = torch.from_numpy(np.ascontiguousarray(np.asarray(point, dtype=np.float64).reshape(1, 3))).to(dev)
    ex = exclude_object_id is not None and exclude_cell is not None
    eo = torch.tensor([int(exclude_object_id)], dtype=torch.int64, device=dev) if ex else None
    ec = torch.tensor([int(exclude_cell)], dtype=torch.int64, device=dev) if ex else None
    tau = torch.empty(1, dtype=torch.float64, device=dev)
    st = torch.zeros(4, dtype=torch.int64, device=dev)
    rc = _lib.load().fhv_transmittance(_lib.ctx(dev), 1, _lib.ptr(p), 0, _lib.ptr(eo), _lib.ptr(ec), _volume(fhv),
                                       sh.struct(), float(cfg.splat_radius_world), float(cfg.shadow_epsilon),
                                       _lib.ptr(tau), _lib.ptr(st), _lib.stream_ptr(dev))
    _lib.check(rc, "shadow_transmittance")
    _merge(stats, st.cpu().tolist(), hits=False)
    return float(tau.item())
