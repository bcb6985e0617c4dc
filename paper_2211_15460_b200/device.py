"""HBM residency of the inputs: triangle arrays, capture configs, shading tables.

Layout in HBM (SURVEY.md section 8(d), 176 B per triangle):
  pos  f64[T,3,3]  72 B   vertex positions
  vnrm f64[T,3,3]  72 B   vertex normals
  fnrm f64[T,3]    24 B   face normals
  mat, obj u32[T]   8 B
f64 is kept on purpose: coverage ties are decided on the reference's f64
edge functions, so inputs must stay bit-identical.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .lights import pack_lights, pack_materials


def default_device(device=None) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("fhv_b200 needs a CUDA device (B200); there is no CPU fallback")
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError("fhv_b200 runs on CUDA devices only")
    return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())


class DeviceScene:
    """Triangle arrays resident on one device (uploaded once per scene)."""

    def __init__(self, scene, device: torch.device, pinned: bool = False):
        def up(a, dt):
            t = torch.from_numpy(np.ascontiguousarray(a)).to(dt)
            if pinned:
                t = t.pin_memory()
            return t.to(device, non_blocking=True)
        self.device = device
        self.n_tri = scene.n_triangles
        self.pos = up(scene.positions, torch.float64)
        self.vnrm = up(scene.normals, torch.float64)
        self.fnrm = up(scene.face_normals, torch.float64)
        self.mat = up(scene.material_id.view(np.int32), torch.int32).view(torch.uint32)
        self.obj = up(scene.object_id.view(np.int32), torch.int32).view(torch.uint32)

    @staticmethod
    def from_tensors(pos, vnrm, fnrm, mat, obj) -> "DeviceScene":
        self = DeviceScene.__new__(DeviceScene)
        self.device = pos.device
        self.n_tri = int(pos.shape[0])
        self.pos, self.vnrm, self.fnrm, self.mat, self.obj = pos, vnrm, fnrm, mat, obj
        return self

    def derive_face_normals(self) -> torch.Tensor:
        """Recompute ``fnrm`` on the device from ``pos`` with make_triangle's
        arithmetic (fhv/scene.py:137-139: cross, sqrt(FWD dot), divide), on the
        current stream.  Bit-identical to the host face normals of any scene
        built by make_triangle (tests/test_gpu_parity.py), so a pipelined
        caller need not upload them."""
        lib = _lib.load()
        rc = lib.fhv_face_normals(_lib.ctx(self.device), self.n_tri, _lib.ptr(self.pos), _lib.ptr(self.fnrm),
                                  _lib.stream_ptr(self.device))
        _lib.check(rc, "face normals")
        return self.fnrm

    def struct(self) -> _lib.Tris:
        # the C struct is cached with the pointers it was built from
        key = (self.n_tri, self.pos.data_ptr(), self.vnrm.data_ptr(), self.fnrm.data_ptr(), self.mat.data_ptr(),
               self.obj.data_ptr())
        hit = self.__dict__.get("_struct")
        if hit is None or hit[0] != key:
            hit = self.__dict__["_struct"] = (key, _lib.Tris(self.n_tri, _lib.ptr(self.pos), _lib.ptr(self.vnrm),
                                                             _lib.ptr(self.fnrm), _lib.ptr(self.mat),
                                                             _lib.ptr(self.obj)))
        return hit[1]

    @property
    def nbytes(self) -> int:
        return 176 * self.n_tri


def device_scene(scene, device=None) -> DeviceScene:
    """Cached upload of a Scene (keyed by device)."""
    dev = default_device(device)
    cache = scene.__dict__.setdefault("_device_cache", {})
    ds = cache.get(str(dev))
    if ds is None:
        ds = DeviceScene(scene, dev)
        cache[str(dev)] = ds
    return ds


def capture_cfg(plan) -> _lib.CaptureCfg:
    c = _lib.CaptureCfg()
    c.strategy = plan.strategy
    c.res = plan.res
    c.pitch = plan.pitch
    flat = np.ascontiguousarray(plan.proj, dtype=np.float64).reshape(48)
    ctypes.memmove(c.proj, flat.ctypes.data, 48 * 8)
    return c


class DeviceShading:
    """Material and light tables on the device (fhv_shading_t)."""

    def __init__(self, materials, lights, device: torch.device):
        md, ms, msh, ma = pack_materials(materials)
        lk, lv, lc, la = pack_lights(lights)

        def up(a, dt=None):
            t = torch.from_numpy(np.ascontiguousarray(a))
            return t.to(device) if dt is None else t.to(dt).to(device)
        self.tensors = [up(lk.astype(np.uint8)), up(lv), up(lc), up(la), up(md), up(ms), up(msh), up(ma)]
        self.n_lights = len(lights)
        self.n_mats = len(md)

    @staticmethod
    def from_arrays(mats: dict, lights, device: torch.device) -> "DeviceShading":
        """From material_arrays()-style tables (the reference's ``mats`` dicts)."""
        self = DeviceShading.__new__(DeviceShading)
        lk, lv, lc, la = pack_lights(lights)
        arrs = [np.ascontiguousarray(np.asarray(mats[k], dtype=np.float64))
                for k in ("diffuse", "specular", "shininess", "alpha")]
        self.tensors = [torch.from_numpy(np.ascontiguousarray(a)).to(device) for a in (lk.astype(np.uint8), lv, lc, la)]
        self.tensors += [torch.from_numpy(a).to(device) for a in arrs]
        self.n_lights = len(lights)
        self.n_mats = len(arrs[3])
        return self

    def struct(self) -> _lib.Shading:
        st = self.__dict__.get("_struct")
        if st is None:  # tables are immutable after construction
            t = self.tensors
            st = self.__dict__["_struct"] = _lib.Shading(
                self.n_lights, _lib.ptr(t[0]), _lib.ptr(t[1]), _lib.ptr(t[2]), _lib.ptr(t[3]), self.n_mats,
                _lib.ptr(t[4]), _lib.ptr(t[5]), _lib.ptr(t[6]), _lib.ptr(t[7]))
        return st


def host_f64(values) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(values, dtype=np.float64))
