"""Capture configuration: raster configs, projections and capture strategies.

Host-side mirror of ``fhv/raster.py``.  Everything here is small f64 setup
computed with the reference's own NumPy expressions (so the 4x4 projection
bits match), packed into a :class:`CapturePlan` that the device rasteriser
consumes.  The per-triangle rasterisation itself (``_raster_screen`` /
``_raster_tangent`` / ``coverage``, fhv/raster.py:184-242 and
fhv/_ckern.pyx:25-105) runs on the GPU, see ``csrc/fhv_capture.cu``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .scene import Camera, Scene, SceneError, capture_camera

__all__ = ["CAPTURE_STRATEGIES", "CapturePlan", "CaptureStats", "CaptureStrategy", "EmittedFragment",
           "FragmentBatch", "ListSink", "capture_pass", "RasterConfig", "capture_plan", "ortho_projection", "perspective_projection",
           "rasterize_triangle", "rasterize_triangles", "tangent_basis", "world_pixel_footprint"]

CAPTURE_STRATEGIES = ("one_view", "three_separate", "three_way_geometry", "normal_space")
STRATEGY_CODE = {k: i for i, k in enumerate(CAPTURE_STRATEGIES)}


def ortho_projection(camera: Camera) -> np.ndarray:
    """World -> clip for an orthographic camera (fhv/raster.py:37-51)."""
    r, u, f = camera.basis()
    hh = camera.extent_or_fov / 2.0
    hw = hh * camera.aspect
    zs = 1.0 / (camera.far - camera.near)
    m = np.zeros((4, 4))
    m[0, :3], m[0, 3] = r / hw, -float(camera.eye @ r) / hw
    m[1, :3], m[1, 3] = u / hh, -float(camera.eye @ u) / hh
    m[2, :3], m[2, 3] = f * zs, -(float(camera.eye @ f) + camera.near) * zs
    m[3, 3] = 1.0
    return m


def perspective_projection(camera: Camera) -> np.ndarray:
    """World -> clip for a perspective camera (fhv/raster.py:54-68)."""
    r, u, f = camera.basis()
    t = math.tan(math.radians(camera.extent_or_fov) / 2.0)
    zs = camera.far / (camera.far - camera.near)
    m = np.zeros((4, 4))
    m[0, :3], m[0, 3] = r / (t * camera.aspect), -float(camera.eye @ r) / (t * camera.aspect)
    m[1, :3], m[1, 3] = u / t, -float(camera.eye @ u) / t
    m[2, :3], m[2, 3] = f * zs, -(float(camera.eye @ f) + camera.near) * zs
    m[3, :3], m[3, 3] = f, -float(camera.eye @ f)
    return m


@dataclass
class RasterConfig:
    """Resolution + projection of one raster pass (fhv/raster.py:71-104)."""

    resolution: tuple
    projection: np.ndarray
    extent: float | None = 1.0
    depth_range: tuple = (0.0, 1.0)
    fill_rule: str = "top-left"

    def __post_init__(self):
        w, h = self.resolution
        if w < 1 or h < 1:
            raise SceneError("raster resolution must be >= 1")
        self.projection = np.asarray(self.projection, dtype=np.float64)
        if self.projection.shape != (4, 4):
            raise SceneError("projection must be 4x4")
        if abs(np.linalg.det(self.projection)) < 1e-30:
            raise SceneError("projection must be invertible")

    @property
    def is_orthographic(self) -> bool:
        return bool(np.array_equal(self.projection[3], (0.0, 0.0, 0.0, 1.0)))

    @staticmethod
    def from_camera(camera: Camera) -> "RasterConfig":
        if camera.kind == "orthographic":
            return RasterConfig(camera.resolution, ortho_projection(camera), extent=camera.extent_or_fov)
        return RasterConfig(camera.resolution, perspective_projection(camera), extent=None)


def world_pixel_footprint(cfg: RasterConfig) -> float:
    if cfg.extent is None:
        raise SceneError("pixel footprint requires an orthographic config")
    return cfg.extent / cfg.resolution[1]


def tangent_basis(n) -> np.ndarray:
    """Rows (t, b, n) for a unit normal (fhv/raster.py:147-163).  Host helper;
    the device computes the same basis per triangle in f64."""
    n = np.asarray(n, dtype=np.float64)
    norm = float(np.linalg.norm(n))
    if norm < 1e-12:
        raise ValueError("tangent_basis: zero-length normal")
    if abs(norm - 1.0) > 1e-3:
        raise ValueError(f"tangent_basis: |n| = {norm}, expected unit")
    n = n / norm
    h = np.array([1.0, 0.0, 0.0]) if abs(n[0]) <= 0.6 else np.array([0.0, 1.0, 0.0])
    t = h - float(h @ n) * n
    t = t / np.linalg.norm(t)
    return np.stack([t, np.cross(n, t), n])


@dataclass
class EmittedFragment:
    """One fragment (fhv/raster.py:114-121): what ppfl_insert / pofl_insert take."""

    raster_xy: tuple
    world_position: np.ndarray
    world_normal: np.ndarray
    depth: float
    material_id: int
    object_id: int


@dataclass
class FragmentBatch:
    """All fragments of one (triangle, pass) job, struct-of-arrays (fhv/raster.py:124-144)."""

    raster_x: np.ndarray
    raster_y: np.ndarray
    world_position: np.ndarray
    world_normal: np.ndarray
    depth: np.ndarray
    material_id: int
    object_id: int

    def __len__(self) -> int:
        return len(self.raster_x)

    def fragments(self):
        for i in range(len(self.raster_x)):
            yield EmittedFragment((int(self.raster_x[i]), int(self.raster_y[i])), self.world_position[i],
                                  self.world_normal[i], float(self.depth[i]), self.material_id, self.object_id)


class ListSink:
    """Collects emitted batches (fhv/raster.py:309-320; test/inspection helper)."""

    def __init__(self):
        self.batches: list = []

    def __call__(self, batch: FragmentBatch) -> None:
        self.batches.append(batch)

    @property
    def total(self) -> int:
        return sum(len(b) for b in self.batches)


@dataclass(frozen=True)
class CaptureStrategy:
    kind: str
    axis: str = "+z"

    def __post_init__(self):
        if self.kind not in CAPTURE_STRATEGIES:
            raise SceneError(f"unknown capture strategy {self.kind!r}")

    @staticmethod
    def one_view(axis: str = "+z") -> "CaptureStrategy":
        return CaptureStrategy("one_view", axis)

    @staticmethod
    def three_separate() -> "CaptureStrategy":
        return CaptureStrategy("three_separate")

    @staticmethod
    def three_way_geometry() -> "CaptureStrategy":
        return CaptureStrategy("three_way_geometry")

    @staticmethod
    def normal_space() -> "CaptureStrategy":
        return CaptureStrategy("normal_space")

    @staticmethod
    def parse(name: str, axis: str = "+z") -> "CaptureStrategy":
        key = name.replace("-", "_")
        key = {"three_way": "three_way_geometry", "normal": "normal_space"}.get(key, key)
        return CaptureStrategy(key, axis)


@dataclass
class CaptureStats:
    fragments_emitted: int = 0
    triangles_processed: int = 0
    passes: int = 0
    draw_batches: int = 0

    def as_dict(self) -> dict:
        return {"fragments_emitted": self.fragments_emitted,
                "triangles_processed": self.triangles_processed,
                "passes": self.passes, "draw_batches": self.draw_batches}


@dataclass
class CapturePlan:
    """Everything the device rasteriser needs besides the triangles.

    strategy : index into CAPTURE_STRATEGIES
    res      : square capture grid edge (fhv/raster.py:359)
    pitch    : tangent-space sample spacing (normal_space)
    proj     : (n_axes, 4, 4) f64 capture projections; job -> axis mapping
               follows fhv/raster.py:366-383
    n_jobs   : number of (triangle, pass) jobs = CaptureStats.triangles_processed
    passes   : CaptureStats.passes
    """

    strategy: int
    res: int
    pitch: float
    proj: np.ndarray
    n_jobs: int
    passes: int
    n_objects: int

    def stats(self, emitted: int) -> CaptureStats:
        return CaptureStats(int(emitted), self.n_jobs, self.passes, self.passes * self.n_objects)


def capture_plan(scene: Scene, strategy: CaptureStrategy, cfg: RasterConfig) -> CapturePlan:
    """Resolve a strategy + config into per-axis projections (fhv/raster.py:350-388)."""
    if cfg.extent is None:
        raise SceneError("capture requires an orthographic config")
    res = int(cfg.resolution[1])
    T = scene.n_triangles

    def axis_proj(axis: str) -> np.ndarray:
        return RasterConfig.from_camera(capture_camera(scene, axis, res)).projection

    code = STRATEGY_CODE[strategy.kind]
    proj = np.zeros((3, 4, 4))
    pitch = 0.0
    if strategy.kind == "one_view":
        proj[0] = axis_proj(strategy.axis)
        n_jobs, passes = T, 1
    elif strategy.kind in ("three_separate", "three_way_geometry"):
        for i, a in enumerate(("+x", "+y", "+z")):
            proj[i] = axis_proj(a)
        n_jobs, passes = 3 * T, (3 if strategy.kind == "three_separate" else 1)
    else:
        pitch = world_pixel_footprint(cfg)
        n_jobs, passes = T, 1
    return CapturePlan(code, res, float(pitch), proj, n_jobs, passes, scene.n_objects)


def rasterize_triangles(scene: Scene, cfg: RasterConfig, device=None) -> dict:
    """``_raster_screen`` of every triangle of ``scene`` through ``cfg`` on the
    device (fhv_raster_screen): fragments in (triangle, y, x) order as CUDA
    tensors ``job`` (triangle index), ``raster_x``, ``raster_y``,
    ``world_position``, ``world_normal``, ``depth``."""
    import ctypes

    import torch

    from . import _lib
    from .device import device_scene, host_f64
    ds = device_scene(scene, device)
    dev = ds.device
    lib = _lib.load()
    cx, st = _lib.ctx(dev), _lib.stream_ptr(dev)
    proj = host_f64(cfg.projection).reshape(16)
    w, h = (int(v) for v in cfg.resolution)
    n = ctypes.c_int64(0)
    rc = lib.fhv_raster_screen(cx, ds.struct(), proj.ctypes.data, w, h, 0, None, None, None, None, None, None,
                               ctypes.byref(n), st)
    _lib.check(rc, "rasterize_triangle")
    m = int(n.value)
    job = torch.empty(m, dtype=torch.int64, device=dev)
    px = torch.empty(m, dtype=torch.int32, device=dev)
    py = torch.empty(m, dtype=torch.int32, device=dev)
    wpos = torch.empty((m, 3), dtype=torch.float64, device=dev)
    wnrm = torch.empty((m, 3), dtype=torch.float64, device=dev)
    dep = torch.empty(m, dtype=torch.float64, device=dev)
    if m:
        rc = lib.fhv_raster_screen(cx, ds.struct(), proj.ctypes.data, w, h, m, _lib.ptr(job), _lib.ptr(px),
                                   _lib.ptr(py), _lib.ptr(wpos), _lib.ptr(wnrm), _lib.ptr(dep), ctypes.byref(n), st)
        _lib.check(rc, "rasterize_triangle")
    return {"job": job, "raster_x": px, "raster_y": py, "world_position": wpos, "world_normal": wnrm, "depth": dep}


def rasterize_triangle(tri, cfg: RasterConfig, sink=None, device=None) -> int:
    """Rasterise one triangle through ``cfg`` (fhv/raster.py:245-252): emits
    one FragmentBatch (host arrays, the reference's types) to ``sink`` when it
    covers any pixel; returns the fragment count."""
    from .scene import Material, Scene
    out = rasterize_triangles(Scene.from_triangles([tri], [Material()] * (int(tri.material_id) + 1)), cfg, device)
    n = int(out["job"].numel())
    if n and sink is not None:
        sink(FragmentBatch(out["raster_x"].cpu().numpy(), out["raster_y"].cpu().numpy(),
                           out["world_position"].cpu().numpy(), out["world_normal"].cpu().numpy(),
                           out["depth"].cpu().numpy(), int(tri.material_id), int(tri.object_id)))
    return n


def capture_pass(scene, strategy: CaptureStrategy, cfg: RasterConfig, sink, threads: int = 1, device=None):
    """fhv.raster.capture_pass (fhv/raster.py:350-388) at its reference module
    path; the implementation is capture.capture_pass (device rasterisation,
    host sink calls)."""
    from .capture import capture_pass as _capture_pass
    return _capture_pass(scene, strategy, cfg, sink, threads, device=device)
