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

    def load_indexed(self, up: "IndexedUpload") -> "DeviceScene":
        """Fill this scene's triangle arrays from indexed device buffers on the
        current stream: the gather (fhv_expand_indexed), the ids, and the face
        normals re-derived with make_triangle's arithmetic."""
        if up.n_tri != self.n_tri:
            raise ValueError("indexed upload has a different triangle count")
        lib = _lib.load()
        rc = lib.fhv_expand_indexed(_lib.ctx(self.device), up.n_vert, _lib.ptr(up.vpos), _lib.ptr(up.vn), up.n_tri,
                                    _lib.ptr(up.faces), _lib.ptr(self.pos), _lib.ptr(self.vnrm),
                                    _lib.stream_ptr(self.device))
        _lib.check(rc, "expand indexed")
        self.mat.view(torch.int32).copy_(up.mat)
        self.obj.view(torch.int32).copy_(up.obj)
        self.derive_face_normals()
        return self

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


class IndexedMesh:
    """A scene's triangle arrays in shared-vertex form, for cheap uploads:
    (position, vertex normal) rows deduplicated by their exact bytes and the
    faces as u32 vertex indices -- the same doubles, ~1/3.5 of the bytes for a
    mesh (each vertex shared by ~6 triangles).  ``DeviceScene.load_indexed``
    expands them on the device into the triangle arrays ``make_triangle`` /
    ``load_scene`` produce (fhv/scene.py:129-146, 291-378), byte for byte;
    face normals are re-derived there (``derive_face_normals``)."""

    def __init__(self, vpos: np.ndarray, vn: np.ndarray, faces: np.ndarray, mat: np.ndarray, obj: np.ndarray):
        self.vpos = np.ascontiguousarray(vpos, dtype=np.float64)
        self.vn = np.ascontiguousarray(vn, dtype=np.float64)
        self.faces = np.ascontiguousarray(faces, dtype=np.uint32)
        self.mat = np.ascontiguousarray(mat, dtype=np.uint32)
        self.obj = np.ascontiguousarray(obj, dtype=np.uint32)
        if self.vpos.shape != self.vn.shape or self.vpos.ndim != 2 or self.vpos.shape[1] != 3:
            raise ValueError("vertex rows must be [n_vert, 3] positions and normals")
        if self.faces.ndim != 2 or self.faces.shape[1] != 3 or len(self.mat) != len(self.faces) \
                or len(self.obj) != len(self.faces):
            raise ValueError("faces must be [n_tri, 3] with one material / object id per face")
        if len(self.faces) and int(self.faces.max()) >= len(self.vpos):
            raise ValueError("face vertex index out of range")

    @staticmethod
    def from_scene(scene) -> "IndexedMesh":
        """Deduplicate a scene's corners (cached on the scene)."""
        hit = scene.__dict__.get("_indexed_mesh")
        if hit is not None:
            return hit
        T = scene.n_triangles
        rows = np.ascontiguousarray(np.concatenate((scene.positions.reshape(3 * T, 3),
                                                    scene.normals.reshape(3 * T, 3)), axis=1))
        keys = rows.view(np.dtype((np.void, 48))).reshape(-1)
        _, first, inv = np.unique(keys, return_index=True, return_inverse=True)
        uniq = rows[first]
        mesh = IndexedMesh(uniq[:, :3], uniq[:, 3:], inv.reshape(T, 3).astype(np.uint32),
                           scene.material_id, scene.object_id)
        scene.__dict__["_indexed_mesh"] = mesh
        return mesh

    @property
    def n_vertices(self) -> int:
        return len(self.vpos)

    @property
    def n_triangles(self) -> int:
        return len(self.faces)

    @property
    def nbytes(self) -> int:
        return self.vpos.nbytes + self.vn.nbytes + self.faces.nbytes + self.mat.nbytes + self.obj.nbytes

    def arrays(self) -> tuple:
        return self.vpos, self.vn, self.faces.view(np.int32), self.mat.view(np.int32), self.obj.view(np.int32)


class IndexedUpload:
    """Device staging buffers of one IndexedMesh (vertex rows, faces, ids),
    refilled by each upload (e.g. from pinned host copies on a copy stream)."""

    def __init__(self, mesh: IndexedMesh, device: torch.device):
        self.n_vert, self.n_tri = mesh.n_vertices, mesh.n_triangles
        self.vpos = torch.empty((self.n_vert, 3), dtype=torch.float64, device=device)
        self.vn = torch.empty((self.n_vert, 3), dtype=torch.float64, device=device)
        self.faces = torch.empty((self.n_tri, 3), dtype=torch.int32, device=device)
        self.mat = torch.empty(self.n_tri, dtype=torch.int32, device=device)
        self.obj = torch.empty(self.n_tri, dtype=torch.int32, device=device)

    def tensors(self) -> tuple:
        return self.vpos, self.vn, self.faces, self.mat, self.obj


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
