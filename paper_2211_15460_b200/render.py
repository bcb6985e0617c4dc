"""Point-splat reconstruction on the device (splat_render, fhv/render.py:249-320).

Also re-exports the shading / compositing value types (see lights.py) so the
module mirrors ``fhv.render``.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .device import DeviceShading, host_f64
from .lights import (GBuffer, ImageBuffer, Light, composite_over, front_to_back_accumulate, headlight,
                     material_arrays, read_float_dump, read_ppm, resolve_over_background, srgb_encode,
                     write_float_dump, write_ppm)
from .scene import Camera, SceneError

__all__ = ["GBuffer", "ImageBuffer", "Light", "composite_over", "deferred_baseline", "front_to_back_accumulate",
           "headlight",
           "material_arrays", "project_points", "read_float_dump", "read_ppm", "resolve_over_background", "shade",
           "shade_many", "splat_render", "srgb_encode", "write_float_dump", "write_ppm"]


def _dev_f64(a, dev, cols: int | None = 3) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        t = a.to(device=dev, dtype=torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to(dev)
    return t.reshape(-1, cols).contiguous() if cols else t.reshape(-1).contiguous()


def shade_many(points, normals, material_id, mats, lights, eye, device=None):
    """Blinn-Phong over fragment arrays, channels clamped to [0, 1]
    (fhv/render.py:120-156), on the device (fhv_shade).  ``mats`` is a
    material_arrays() dict or a list of Materials.  NumPy inputs give a
    NumPy (n, 3) result, CUDA tensors a CUDA tensor."""
    from .device import default_device
    on_dev = isinstance(points, torch.Tensor) and points.is_cuda
    dev = points.device if on_dev else default_device(device)
    p = _dev_f64(points, dev)
    q = _dev_f64(normals, dev)
    m = (material_id.to(device=dev, dtype=torch.int64) if isinstance(material_id, torch.Tensor)
         else torch.from_numpy(np.ascontiguousarray(np.atleast_1d(np.asarray(material_id)).astype(np.int64))).to(dev))
    m = m.reshape(-1).contiguous()
    n = p.shape[0]
    if q.shape[0] != n or m.numel() != n:
        raise ValueError("shade_many: points, normals and material_id disagree in length")
    sh = DeviceShading.from_arrays(mats, lights, dev) if isinstance(mats, dict) else DeviceShading(mats, lights, dev)
    if n and (int(m.min()) < 0 or int(m.max()) >= sh.n_mats):
        raise IndexError("shade_many: material id outside the material table")
    out = torch.empty((n, 3), dtype=torch.float64, device=dev)
    e = host_f64(eye.cpu() if isinstance(eye, torch.Tensor) else eye).reshape(3)
    rc = _lib.load().fhv_shade(_lib.ctx(dev), n, _lib.ptr(p), _lib.ptr(q), _lib.ptr(m), sh.n_mats, sh.struct(),
                               e.ctypes.data, _lib.ptr(out), _lib.stream_ptr(dev))
    _lib.check(rc, "shade_many")
    return out if on_dev else out.cpu().numpy()


def shade(position, normal, material, light, eye, device=None) -> np.ndarray:
    """Blinn-Phong for a single fragment and light (fhv/render.py:159-165)."""
    return shade_many(np.asarray(position, dtype=np.float64), np.asarray(normal, dtype=np.float64), np.array([0]),
                      material_arrays([material]), [light], np.asarray(eye, dtype=np.float64), device)[0]


def project_points(camera: Camera, points, device=None):
    """Raster coordinates, [0, 1] depth and view distance of world points
    (fhv/render.py:211-233), on the device (fhv_project_points): returns
    (xr, yr, depth, zc) like the reference (NumPy in, NumPy out)."""
    from .device import default_device
    on_dev = isinstance(points, torch.Tensor) and points.is_cuda
    dev = points.device if on_dev else default_device(device)
    one_d = np.ndim(points) == 1 if not on_dev else points.dim() == 1
    p = _dev_f64(points, dev)
    n = p.shape[0]
    outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(4)]
    cam = host_f64(camera.scalars())
    rc = _lib.load().fhv_project_points(_lib.ctx(dev), n, _lib.ptr(p), cam.ctypes.data, *[_lib.ptr(o) for o in outs],
                                        _lib.stream_ptr(dev))
    _lib.check(rc, "project_points")
    if on_dev:
        return tuple(o[0] if one_d else o for o in outs)
    res = [o.cpu().numpy() for o in outs]
    return tuple(float(r[0]) if one_d else r for r in res)


def splat_render(pool, camera: Camera, lights, splat_radius_world: float, materials,
                 background=(0.0, 0.0, 0.0, 0.0), id_buffer: GBuffer | None = None, *,
                 packed: bool = False, n: int | None = None, out: ImageBuffer | None = None,
                 shading: DeviceShading | None = None) -> ImageBuffer:
    """Z-tested point splatting of a fragment pool into a novel view.

    Returns an ImageBuffer whose ``pixels`` (h, w, 4) and ``depth`` (h, w)
    are float64 CUDA tensors.  ``id_buffer`` (GBuffer of CUDA tensors, e.g.
    from :func:`device_gbuffer`) receives the winners' attributes.
    ``packed=True`` selects the single 64-bit (f32 depth | index) atomicMin
    variant.  ``out`` reuses preallocated image tensors; ``shading`` a
    prebuilt DeviceShading (materials + lights already on the device).
    """
    if splat_radius_world <= 0.0:
        raise SceneError("splat radius must be > 0")
    dev = pool.device
    w, h = camera.resolution
    if out is None:
        out = ImageBuffer(w, h, torch.empty((h, w, 4), dtype=torch.float64, device=dev),
                          torch.empty((h, w), dtype=torch.float64, device=dev))
    count = pool.stored_count if n is None else int(n)
    if shading is None:
        shading = DeviceShading(materials, lights, dev)
    gb = None
    if id_buffer is not None:
        gb = _lib.GBuf(_lib.ptr(id_buffer.position), _lib.ptr(id_buffer.normal), _lib.ptr(id_buffer.material_id),
                       _lib.ptr(id_buffer.object_id), _lib.ptr(id_buffer.valid))
    cam = host_f64(camera.scalars())
    bg = host_f64(background)
    flags = _lib.FHV_SPLAT_PACKED if packed else 0
    if getattr(pool, "in_unit_cube", False) and footprint_bounded(camera, float(splat_radius_world)):
        flags |= _lib.FHV_SPLAT_NOSYNC  # SceneError impossible: no need to wait for the kernels
    lib = _lib.load()
    rc = lib.fhv_splat(_lib.ctx(dev), count, _lib.ptr(pool.position), _lib.ptr(pool.normal),
                       _lib.ptr(pool.material_id), _lib.ptr(pool.object_id), cam.ctypes.data, float(splat_radius_world),
                       bg.ctypes.data, shading.struct(), _lib.ptr(out.pixels), _lib.ptr(out.depth), None,
                       gb, flags, _lib.stream_ptr(dev))
    _lib.check(rc, "splat_render")
    return out


_UNIT_LO, _UNIT_HI = -1e-6, 1.0 + 1e-6  # cell_code's accepted range (fhv/storage.py:152-155)


def footprint_bounded(camera: Camera, radius: float) -> bool:
    """True when NO point of [-1e-6, 1+1e-6]^3 can get a splat footprint over
    the reference's 4096-pixel limit (fhv/render.py:285-286) -- then the
    device-side check (and its sync) is unnecessary.  Orthographic: the
    half-size is a constant.  Perspective: half = r h / (2 tan zc) decreases
    with the view depth zc, bounded below over the cube by its nearest corner
    (points with zc <= 1e-9 are not drawn)."""
    key = (camera.scalars().tobytes(), radius)
    hit = camera.__dict__.get("_fp_bound")
    if hit is not None and hit[0] == key:
        return hit[1]
    c = camera.scalars()
    h = c[14]
    if c[0] == 0.0:
        half = radius * h / c[21]
    else:
        f, eye = c[10:13], c[1:4]
        zmin = sum(min(_UNIT_LO * fa, _UNIT_HI * fa) for fa in f) - float(eye @ f)
        zmin -= 1e-9 * (1.0 + abs(zmin))  # slack for the device's rounding of zc
        half = float("inf") if zmin <= 1e-9 else radius * h / ((2.0 * c[17]) * zmin) * (1.0 + 1e-9)
    ok = bool((2.0 * max(half, 0.5) + 2.0) ** 2 <= 4096.0)
    camera.__dict__["_fp_bound"] = (key, ok)
    return ok


def deferred_baseline(scene, camera: Camera, lights, background=(0.0, 0.0, 0.0, 0.0), *, device=None,
                      tris=None, shading: DeviceShading | None = None, out=None):
    """Two-phase reference renderer (fhv/render.py:327-382) on the device:
    depth-tested geometry pass into a G-buffer (nearest f64 depth per pixel,
    equal depths keep the earlier triangle), then one shading pass.

    Returns ``(ImageBuffer, GBuffer)`` of CUDA tensors with the reference's
    dtypes (f64 pixels / depth / position / normal, int32 ids, bool valid).
    ``tris``: a DeviceScene already holding the scene; ``shading``: prebuilt
    DeviceShading; ``out``: a previous ``(ImageBuffer, GBuffer)`` to reuse.
    """
    from .device import device_scene
    from .raster import RasterConfig
    ds = tris if tris is not None else device_scene(scene, device)
    dev = ds.device
    w, h = camera.resolution
    if out is None:
        img = ImageBuffer(w, h, torch.empty((h, w, 4), dtype=torch.float64, device=dev),
                          torch.empty((h, w), dtype=torch.float64, device=dev))
        gb = GBuffer(torch.empty((h, w, 3), dtype=torch.float64, device=dev),
                     torch.empty((h, w, 3), dtype=torch.float64, device=dev),
                     torch.empty((h, w), dtype=torch.int32, device=dev),
                     torch.empty((h, w), dtype=torch.int32, device=dev),
                     torch.empty((h, w), dtype=torch.bool, device=dev))
    else:
        img, gb = out
    if shading is None:
        shading = DeviceShading(scene.materials, lights, dev)
    proj = host_f64(RasterConfig.from_camera(camera).projection).reshape(16)
    eye = host_f64(camera.eye)
    bg = host_f64(background)
    g = _lib.GBuf(_lib.ptr(gb.position), _lib.ptr(gb.normal), _lib.ptr(gb.material_id), _lib.ptr(gb.object_id),
                  _lib.ptr(gb.valid))
    import ctypes
    n = ctypes.c_int64(0)
    lib = _lib.load()
    rc = lib.fhv_deferred(_lib.ctx(dev), ds.struct(), proj.ctypes.data, int(w), int(h), eye.ctypes.data,
                          shading.struct(), bg.ctypes.data, _lib.ptr(img.pixels), _lib.ptr(img.depth), g,
                          ctypes.byref(n), _lib.stream_ptr(dev))
    _lib.check(rc, "deferred_baseline")
    return img, gb


def device_gbuffer(width: int, height: int, device) -> GBuffer:
    """GBuffer of CUDA tensors for splat_render's id_buffer."""
    return GBuffer(torch.zeros((height, width, 3), dtype=torch.float64, device=device),
                   torch.zeros((height, width, 3), dtype=torch.float64, device=device),
                   torch.full((height, width), -1, dtype=torch.int32, device=device),
                   torch.full((height, width), -1, dtype=torch.int32, device=device),
                   torch.zeros((height, width), dtype=torch.uint8, device=device))


def image_numpy(img: ImageBuffer) -> ImageBuffer:
    """Host copy with the reference's numpy dtypes."""
    px = img.pixels.cpu().numpy() if isinstance(img.pixels, torch.Tensor) else np.asarray(img.pixels)
    dp = img.depth.cpu().numpy() if isinstance(img.depth, torch.Tensor) else np.asarray(img.depth)
    return ImageBuffer(img.width, img.height, px, dp)
