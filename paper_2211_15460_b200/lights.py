"""Lights, image buffers and compositing helpers (host side).

Mirrors the small value types of ``fhv/render.py:37-204``.  These are inputs
and outputs of the device kernels, packed into flat f64 arrays by
:func:`pack_lights` / :func:`pack_materials`.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .scene import Camera, Material, SceneError

__all__ = ["GBuffer", "ImageBuffer", "Light", "composite_over", "front_to_back_accumulate",
           "headlight", "material_arrays", "pack_lights", "pack_materials", "read_float_dump",
           "read_ppm", "resolve_over_background", "srgb_encode", "write_float_dump", "write_ppm"]


@dataclass
class Light:
    """Directional (``direction`` points toward the light) or point light
    with its own ambient term (fhv/render.py:37-65)."""

    kind: str = "directional"
    direction: np.ndarray | None = None
    position: np.ndarray | None = None
    color: tuple = (1.0, 1.0, 1.0)
    ambient: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        if self.kind == "directional":
            if self.direction is None:
                raise SceneError("directional light needs a direction")
            d = np.asarray(self.direction, dtype=np.float64)
            length = float(np.linalg.norm(d))
            if length == 0.0:
                raise SceneError("zero light direction")
            self.direction = d / length
        elif self.kind == "point":
            if self.position is None:
                raise SceneError("point light needs a position")
            self.position = np.asarray(self.position, dtype=np.float64)
        else:
            raise SceneError(f"unknown light kind {self.kind!r}")


def headlight(camera: Camera, color=(1.0, 1.0, 1.0), ambient=(0.1, 0.1, 0.1)) -> Light:
    return Light("directional", direction=-camera.view_dir, color=color, ambient=ambient)


@dataclass
class ImageBuffer:
    width: int
    height: int
    pixels: np.ndarray  # (h, w, 4) float64 linear rgb + alpha
    depth: np.ndarray   # (h, w) float64, +inf where empty

    @staticmethod
    def new(width: int, height: int, background=(0.0, 0.0, 0.0, 0.0)) -> "ImageBuffer":
        px = np.empty((height, width, 4))
        px[:] = np.asarray(background, dtype=np.float64)
        return ImageBuffer(width, height, px, np.full((height, width), np.inf))


@dataclass
class GBuffer:
    position: np.ndarray
    normal: np.ndarray
    material_id: np.ndarray
    object_id: np.ndarray
    valid: np.ndarray

    @staticmethod
    def new(width: int, height: int) -> "GBuffer":
        return GBuffer(np.zeros((height, width, 3)), np.zeros((height, width, 3)),
                       np.full((height, width), -1, dtype=np.int32),
                       np.full((height, width), -1, dtype=np.int32),
                       np.zeros((height, width), dtype=bool))


def material_arrays(materials) -> dict:
    return {"diffuse": np.array([m.diffuse for m in materials], dtype=np.float64).reshape(-1, 3),
            "specular": np.array([m.specular for m in materials], dtype=np.float64).reshape(-1, 3),
            "shininess": np.array([m.shininess for m in materials], dtype=np.float64),
            "alpha": np.array([m.alpha for m in materials], dtype=np.float64)}


def pack_materials(materials) -> tuple:
    """(diffuse[M,3], specular[M,3], shininess[M], alpha[M]) contiguous f64."""
    m = material_arrays(materials or [Material()])
    return tuple(np.ascontiguousarray(m[k]) for k in ("diffuse", "specular", "shininess", "alpha"))


def pack_lights(lights) -> tuple:
    """(kind u8[K], vec f64[K,3], color f64[K,3], ambient f64[K,3]) as in
    fhv/raycast.py:460-466: vec is the direction or the position."""
    K = len(lights)
    kind = np.array([0 if l.kind == "directional" else 1 for l in lights], dtype=np.uint8)
    vec = np.array([l.direction if l.kind == "directional" else l.position for l in lights],
                   dtype=np.float64).reshape(K, 3)
    color = np.array([l.color for l in lights], dtype=np.float64).reshape(K, 3)
    amb = np.array([l.ambient for l in lights], dtype=np.float64).reshape(K, 3)
    return kind, np.ascontiguousarray(vec), np.ascontiguousarray(color), np.ascontiguousarray(amb)


def composite_over(front, back) -> np.ndarray:
    """Straight-alpha Porter-Duff over (fhv/render.py:172-181)."""
    f = np.asarray(front, dtype=np.float64)
    b = np.asarray(back, dtype=np.float64)
    a = f[3] + (1.0 - f[3]) * b[3]
    if a == 0.0:
        return np.zeros(4)
    rgb = (f[3] * f[:3] + (1.0 - f[3]) * b[3] * b[:3]) / a
    return np.array([rgb[0], rgb[1], rgb[2], a])


def front_to_back_accumulate(state, rgba_next) -> np.ndarray:
    s = np.asarray(state, dtype=np.float64).copy()
    n = np.asarray(rgba_next, dtype=np.float64)
    t = (1.0 - s[3]) * n[3]
    s[:3] += t * n[:3]
    s[3] += t
    return s


def resolve_over_background(state, background) -> np.ndarray:
    bg = np.asarray(background, dtype=np.float64)
    out = np.empty(4)
    out[:3] = state[:3] + (1.0 - state[3]) * bg[3] * bg[:3]
    out[3] = state[3] + (1.0 - state[3]) * bg[3]
    return out


def srgb_encode(linear: np.ndarray) -> np.ndarray:
    c = np.clip(linear, 0.0, 1.0)
    enc = np.where(c <= 0.0031308, 12.92 * c, 1.055 * np.power(c, 1.0 / 2.4) - 0.055)
    return np.rint(enc * 255.0).astype(np.uint8)


def write_ppm(image: ImageBuffer, path) -> None:
    data = srgb_encode(np.asarray(image.pixels)[:, :, :3])
    with open(path, "wb") as fh:
        fh.write(f"P6\n{image.width} {image.height}\n255\n".encode("ascii"))
        fh.write(data.tobytes())


def write_float_dump(image: ImageBuffer, path) -> None:
    with open(path, "wb") as fh:
        fh.write(np.array([image.width, image.height], dtype="<u4").tobytes())
        fh.write(np.asarray(image.pixels).astype("<f4").tobytes())


def read_float_dump(path) -> np.ndarray:
    blob = open(path, "rb").read()
    w, h = np.frombuffer(blob, dtype="<u4", count=2)
    return np.frombuffer(blob, dtype="<f4", offset=8).reshape(int(h), int(w), 4)


def read_ppm(path) -> np.ndarray:
    with open(path, "rb") as fh:
        if fh.readline().strip() != b"P6":
            raise ValueError("not a binary PPM")
        w, h = (int(v) for v in fh.readline().split())
        if fh.readline().strip() != b"255":
            raise ValueError("unsupported max value")
        return np.frombuffer(fh.read(w * h * 3), dtype=np.uint8).reshape(h, w, 3)
