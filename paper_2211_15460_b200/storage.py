"""Fragment stores on the device: PPFL, POFL and POFA.

Drop-in for ``fhv/storage.py``: same builder names and signatures
(``build_ppfl``, ``build_pofl``, ``pofa_build``), same volume types
(``FhvPpfl``, ``FhvPofl``, ``FhvPofa``) and pool/directory fields, but every
array is a CUDA tensor written by the sm_100a capture kernels
(``csrc/fhv_capture.cu``) through the C ABI.  ``threads`` is accepted and
ignored (the reference's GIL-bound thread pool has no analogue here).

Pool order: by default fragment k of the reference's sequential emission
order lands at pool index k (``alloc="ordered"``), so pools are bit-identical
to the reference.  Linked-list chains are linked with atomicExch and are
multiset-equal per key; ``exact_order=True`` additionally restores the
reference's chain order (and, for POFA, the in-leaf order), making every
array bit-identical.  ``alloc="atomic"`` is the paper's GPU allocator
(warp-aggregated atomicAdd on one counter): nondeterministic order.
"""
from __future__ import annotations

import ctypes
import struct
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import capture_cfg, default_device, device_scene
from .raster import CaptureStats, CaptureStrategy, RasterConfig, capture_plan
from .scene import Scene

__all__ = [
    "FhvError", "FhvPofa", "FhvPofl", "FhvPpfl", "FragmentPool", "FragmentRecord", "MAX_LEVELS",
    "OccupancyPyramid", "PixelDirectory", "PofaBuildError", "PofaDirectory", "PofaWriteSink", "PoflDirectory",
    "PoflSink", "PpflSink", "CountingSink", "RECORD_DTYPE", "RECORD_SIZE_ALIGNED", "RECORD_SIZE_PACKED",
    "build_pofl", "build_ppfl", "cell_box", "cell_code", "cell_of", "chain_indices", "load_snapshot",
    "memory_report", "morton_decode", "morton_encode", "pofa_build", "pofl_insert", "ppfl_insert",
    "rebuild_pofl_as_pofa", "save_snapshot", "snapshot_bytes",
]

_alloc_lock = threading.Lock()

MAX_LEVELS = 20
RECORD_DTYPE = np.dtype([("position", "<f4", (3,)), ("normal", "<f4", (3,)), ("material_id", "<u4"),
                         ("object_id", "<u4"), ("prev_index", "<i4")])
RECORD_SIZE_PACKED = 36
RECORD_SIZE_ALIGNED = 48


class FhvError(ValueError):
    """Invalid storage parameters or corrupted structure (fhv/storage.py:69-70)."""


class PofaBuildError(FhvError):
    """The two capture passes of an array build disagreed (fhv/storage.py:73-74)."""


# ---------------------------------------------------------------------------
# Morton codes and cells (host utilities, fhv/storage.py:83-172)

_U = np.uint64


def _spread(v):
    v = v & _U(0x1FFFFF)
    for sh, m in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                  (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
        v = (v | (v << _U(sh))) & _U(m)
    return v


def _compact(v):
    v = v & _U(0x1249249249249249)
    for sh, m in ((2, 0x10C30C30C30C30C3), (4, 0x100F00F00F00F00F), (8, 0x1F0000FF0000FF),
                  (16, 0x1F00000000FFFF), (32, 0x1FFFFF)):
        v = (v | (v >> _U(sh))) & _U(m)
    return v


def _check_levels(levels: int) -> None:
    if not 0 <= levels <= MAX_LEVELS:
        raise FhvError(f"levels {levels} outside [0, {MAX_LEVELS}]")


def morton_encode(x, y, z, levels: int):
    _check_levels(levels)
    scalar = np.isscalar(x) and np.isscalar(y) and np.isscalar(z)
    xyz = [np.asarray(v, dtype=np.int64) for v in (x, y, z)]
    side = np.int64(1) << levels
    for name, v in zip("xyz", xyz):
        if np.any(v < 0) or np.any(v >= side):
            raise FhvError(f"{name} cell index outside [0, 2^{levels})")
    code = (_spread(xyz[0].astype(_U)) | (_spread(xyz[1].astype(_U)) << _U(1))
            | (_spread(xyz[2].astype(_U)) << _U(2))).astype(np.int64)
    return int(code) if scalar else code


def morton_decode(code, levels: int):
    _check_levels(levels)
    scalar = np.isscalar(code)
    c = np.asarray(code, dtype=np.int64)
    if np.any(c < 0) or np.any(c >= (np.int64(1) << (3 * levels))):
        raise FhvError(f"code outside [0, 8^{levels})")
    u = c.astype(_U)
    out = tuple(_compact(u >> _U(k)).astype(np.int64) for k in range(3))
    return tuple(int(v) for v in out) if scalar else out


def cell_of(position, levels: int) -> np.ndarray:
    _check_levels(levels)
    p = np.asarray(position, dtype=np.float64)
    if not np.all(np.isfinite(p)):
        raise FhvError("non-finite position")
    if np.any(p < -1e-6) or np.any(p > 1.0 + 1e-6):
        raise FhvError("position outside [0,1]^3")
    side = np.int64(1) << levels
    return np.clip(np.floor(p * float(side)).astype(np.int64), 0, side - 1)


def cell_code(position, levels: int):
    idx = cell_of(position, levels)
    return morton_encode(idx[..., 0], idx[..., 1], idx[..., 2], levels)


def cell_box(code: int, level: int):
    x, y, z = morton_decode(int(code), level)
    size = 1.0 / (1 << level)
    lo = np.array([x, y, z], dtype=np.float64) * size
    return lo, lo + size


# ---------------------------------------------------------------------------
# pool and directories (device tensors)


@dataclass
class FragmentRecord:
    position: np.ndarray
    normal: np.ndarray
    material_id: int
    object_id: int
    prev_index: int


class FragmentPool:
    """Pre-allocated fragment storage, struct-of-arrays on the device
    (fhv/storage.py:188-248).  ``next_free`` keeps counting past capacity;
    records beyond it are dropped and ``overflowed`` is set."""

    def __init__(self, capacity: int, device=None, fill_prev: bool = True):
        if capacity < 0:
            raise FhvError("capacity must be >= 0")
        dev = default_device(device)
        self.capacity = int(capacity)
        self.device = dev
        # one allocation carved into the five SoA arrays (each 256-B aligned)
        c = self.capacity
        sizes = [12 * c, 12 * c, 4 * c, 4 * c, 4 * c]
        offs, o = [], 0
        for b in sizes:
            offs.append(o)
            o += (b + 255) // 256 * 256
        buf = torch.empty(max(o, 1), dtype=torch.uint8, device=dev)
        seg = [buf[a:a + b] for a, b in zip(offs, sizes)]
        self.position = seg[0].view(torch.float32).view(c, 3)
        self.normal = seg[1].view(torch.float32).view(c, 3)
        self.material_id = seg[2].view(torch.uint32)
        self.object_id = seg[3].view(torch.uint32)
        self.prev_index = seg[4].view(torch.int32)
        if fill_prev:
            self.prev_index.fill_(-1)
        self.next_free = 0
        self.overflowed = False
        # every stored position passed cell_code's [-1e-6, 1+1e-6]^3 check (POFL / POFA
        # builds): lets splat_render bound the footprint on the host
        self.in_unit_cube = False

    def narrow(self, n: int) -> "FragmentPool":
        """The first ``n`` records as a pool of capacity ``n`` (views, no copy)."""
        if not 0 <= n <= self.capacity:
            raise FhvError(f"cannot narrow a pool of {self.capacity} records to {n}")
        out = FragmentPool.__new__(FragmentPool)
        out.capacity, out.device = int(n), self.device
        out.position, out.normal = self.position[:n], self.normal[:n]
        out.material_id, out.object_id, out.prev_index = self.material_id[:n], self.object_id[:n], self.prev_index[:n]
        out.next_free = min(self.next_free, n)
        out.overflowed = False
        out.in_unit_cube = self.in_unit_cube
        return out

    def alloc_block(self, n: int) -> int:
        """Reserve n slots (fhv/storage.py:207-213): returns the first index;
        the counter keeps counting past capacity and sets ``overflowed``."""
        with _alloc_lock:
            start = self.next_free
            self.next_free += int(n)
            if self.next_free > self.capacity:
                self.overflowed = True
            return start

    @property
    def stored_count(self) -> int:
        return min(self.next_free, self.capacity)

    def struct(self) -> _lib.Pool:
        return _lib.Pool(self.capacity, _lib.ptr(self.position), _lib.ptr(self.normal), _lib.ptr(self.material_id),
                         _lib.ptr(self.object_id), _lib.ptr(self.prev_index))

    def numpy(self) -> dict:
        """Host copies of the stored prefix (reference dtypes)."""
        n = self.stored_count
        return {"position": self.position[:n].cpu().numpy(), "normal": self.normal[:n].cpu().numpy(),
                "material_id": self.material_id[:n].cpu().numpy(), "object_id": self.object_id[:n].cpu().numpy(),
                "prev_index": self.prev_index[:n].cpu().numpy()}

    def record(self, i: int) -> FragmentRecord:
        if not 0 <= i < self.stored_count:
            raise FhvError(f"record index {i} out of range")
        return FragmentRecord(self.position[i].cpu().numpy(), self.normal[i].cpu().numpy(),
                              int(self.material_id[i]), int(self.object_id[i]), int(self.prev_index[i]))

    def to_struct_array(self) -> np.ndarray:
        h = self.numpy()
        out = np.empty(self.stored_count, dtype=RECORD_DTYPE)
        for k in RECORD_DTYPE.names:
            out[k] = h[k]
        return out

    @staticmethod
    def from_struct_array(arr: np.ndarray, device=None) -> "FragmentPool":
        pool = FragmentPool(len(arr), device)
        pool.position.copy_(torch.from_numpy(np.ascontiguousarray(arr["position"])))
        pool.normal.copy_(torch.from_numpy(np.ascontiguousarray(arr["normal"])))
        pool.material_id.copy_(torch.from_numpy(np.ascontiguousarray(arr["material_id"]).view(np.int32)).view(torch.uint32))
        pool.object_id.copy_(torch.from_numpy(np.ascontiguousarray(arr["object_id"]).view(np.int32)).view(torch.uint32))
        pool.prev_index.copy_(torch.from_numpy(np.ascontiguousarray(arr["prev_index"])))
        pool.next_free = len(arr)
        return pool


@dataclass
class PixelDirectory:
    width: int
    height: int
    heads: torch.Tensor  # int32 (h*w,), -1 = empty

    @staticmethod
    def empty(width: int, height: int, device=None) -> "PixelDirectory":
        return PixelDirectory(width, height, torch.full((width * height,), -1, dtype=torch.int32,
                                                        device=default_device(device)))

    def head(self, x: int, y: int) -> int:
        return int(self.heads[y * self.width + x])


@dataclass
class PoflDirectory:
    levels: int
    heads: torch.Tensor  # int32 (8^L,)

    @staticmethod
    def empty(levels: int, device=None) -> "PoflDirectory":
        _check_levels(levels)
        return PoflDirectory(levels, torch.full((8 ** levels,), -1, dtype=torch.int32, device=default_device(device)))


@dataclass
class PofaDirectory:
    levels: int
    offsets: torch.Tensor  # uint32 (8^L,)
    counts: torch.Tensor   # uint32 (8^L,)


def _pyr_offsets(L: int):
    return [((1 << (3 * k)) - 1) // 7 for k in range(L + 1)]


class OccupancyPyramid:
    """Levels 0..L-1 of 8-bit child masks, stored concatenated on the device
    (the layout the ray-cast kernel reads, fhv/raycast.py:539-544)."""

    def __init__(self, leaf_levels: int, data: torch.Tensor | None = None, device=None):
        _check_levels(leaf_levels)
        if leaf_levels < 1:
            raise FhvError("octree needs at least one level")
        self.leaf_levels = leaf_levels
        n = _pyr_offsets(leaf_levels)[-1]
        if data is None:
            data = torch.zeros(n, dtype=torch.uint8, device=default_device(device))
        self.data = data

    @staticmethod
    def uninitialized(leaf_levels: int, device) -> "OccupancyPyramid":
        """For a kernel that writes every level (the POFA directory pass)."""
        _check_levels(leaf_levels)
        return OccupancyPyramid(leaf_levels, torch.empty(_pyr_offsets(leaf_levels)[-1], dtype=torch.uint8,
                                                         device=device))

    @property
    def levels(self) -> list:
        off = _pyr_offsets(self.leaf_levels)
        return [self.data[off[k]:off[k + 1]] for k in range(self.leaf_levels)]

    def mask(self, level: int, node: int) -> int:
        return int(self.data[_pyr_offsets(self.leaf_levels)[level] + node])

    def set_paths(self, codes) -> None:
        """Mark the root paths of leaf codes occupied (fhv/storage.py:294-301), on the device."""
        dev = self.data.device
        c = (codes.to(device=dev, dtype=torch.int64) if isinstance(codes, torch.Tensor)
             else torch.from_numpy(np.ascontiguousarray(np.atleast_1d(np.asarray(codes, dtype=np.int64)))).to(dev))
        c = c.reshape(-1).contiguous()
        rc = _lib.load().fhv_set_paths(_lib.ctx(dev), self.leaf_levels, c.numel(), _lib.ptr(c), _lib.ptr(self.data),
                                       _lib.stream_ptr(dev))
        if rc == _lib.FHV_BAD_ARGS:
            raise FhvError("set_paths: leaf code outside [0, 8^levels)")
        _lib.check(rc, "set_paths")

    @staticmethod
    def from_leaf_occupancy(occupied, leaf_levels: int, device=None) -> "OccupancyPyramid":
        """Bottom-up masks from a leaf occupancy vector (fhv/storage.py:316-328)."""
        _check_levels(leaf_levels)
        if leaf_levels < 1:
            raise FhvError("octree needs at least one level")
        if isinstance(occupied, torch.Tensor) and occupied.is_cuda:
            dev = occupied.device
            occ = occupied.to(torch.bool).to(torch.uint8).reshape(-1).contiguous()
        else:
            dev = default_device(device)
            occ = torch.from_numpy(np.ascontiguousarray(np.asarray(occupied, dtype=bool).reshape(-1))).to(dev)
            occ = occ.to(torch.uint8)
        if occ.numel() != 8 ** leaf_levels:
            raise FhvError("occupancy length != 8^levels")
        pyr = OccupancyPyramid.uninitialized(leaf_levels, dev)
        rc = _lib.load().fhv_pyramid_from_occupancy(_lib.ctx(dev), leaf_levels, _lib.ptr(occ), _lib.ptr(pyr.data),
                                                    _lib.stream_ptr(dev))
        _lib.check(rc, "from_leaf_occupancy")
        return pyr

    def leaf_occupancy(self) -> torch.Tensor:
        last = self.levels[-1].to(torch.int32)
        bits = (last[:, None] >> torch.arange(8, device=last.device, dtype=torch.int32)) & 1
        return bits.bool().reshape(-1)

    def occupied_leaves(self) -> torch.Tensor:
        return torch.nonzero(self.leaf_occupancy()).reshape(-1).to(torch.int64)

    def equals(self, other: "OccupancyPyramid") -> bool:
        return self.leaf_levels == other.leaf_levels and bool(torch.equal(self.data.cpu(), other.data.cpu()))


# ---------------------------------------------------------------------------
# built volumes


@dataclass
class FhvPpfl:
    directory: PixelDirectory
    pool: FragmentPool
    capture_resolution: int
    stats: CaptureStats | None = None
    materials: list | None = None
    layout = "PPFL"

    def pixel_indices(self, x: int, y: int) -> np.ndarray:
        return _chain(self.directory.heads, self.pool.prev_index, y * self.directory.width + x)


@dataclass
class FhvPofl:
    directory: PoflDirectory
    pyramid: OccupancyPyramid
    pool: FragmentPool
    capture_resolution: int
    stats: CaptureStats | None = None
    materials: list | None = None
    layout = "POFL"

    @property
    def levels(self) -> int:
        return self.directory.levels

    def leaf_indices(self, code: int) -> np.ndarray:
        return _chain(self.directory.heads, self.pool.prev_index, code)

    def occupied_leaves(self) -> torch.Tensor:
        return torch.nonzero(self.directory.heads >= 0).reshape(-1).to(torch.int64)

    pending = None  # (ticket, guessed total, synchronous rebuild) of an asynchronous build_pofl
    done = None     # CUDA event recorded after the asynchronous build's ticket copy

    def wait(self) -> "FhvPofl":
        """Finish an asynchronous build_pofl: synchronise, check its ticket,
        rebuild synchronously in place if the speculation was wrong."""
        if self.pending is None:
            return self
        tk, guess, rebuild = self.pending
        if self.done is not None:
            self.done.synchronize()
        else:
            torch.cuda.current_stream(self.pool.device).synchronize()
        rc = ticket_status(tk, guess)
        self.pending = None
        if rc == _lib.FHV_STALE:
            fresh = rebuild()
            self.directory, self.pyramid, self.pool, self.stats = fresh.directory, fresh.pyramid, fresh.pool, fresh.stats
        else:
            _lib.check(rc, "build_pofl")
        return self


@dataclass
class FhvPofa:
    directory: PofaDirectory
    pyramid: OccupancyPyramid
    pool: FragmentPool
    capture_resolution: int
    stats: CaptureStats | None = None
    materials: list | None = None
    layout = "POFA"

    @property
    def levels(self) -> int:
        return self.directory.levels

    def leaf_indices(self, code: int) -> np.ndarray:
        off = int(self.directory.offsets[code])
        return np.arange(off, off + int(self.directory.counts[code]), dtype=np.int64)

    pending = None  # (ticket, guessed total, synchronous rebuild) of an asynchronous pofa_build
    done = None     # CUDA event recorded after the asynchronous build's ticket copy

    def wait(self) -> "FhvPofa":
        """Finish an asynchronous build: synchronise, check its ticket, and
        rebuild synchronously in place if the speculation was wrong.  Raises
        the build's own error otherwise."""
        if self.pending is None:
            return self
        if self.done is not None:  # the build's stream, whichever stream is current now
            self.done.synchronize()
        else:
            torch.cuda.current_stream(self.pool.device).synchronize()
        rc = check_ticket(self)
        rebuild = self.pending[2]
        self.pending = None
        if rc == _lib.FHV_STALE:
            fresh = rebuild()
            self.directory, self.pyramid, self.pool, self.stats = fresh.directory, fresh.pyramid, fresh.pool, fresh.stats
        else:
            _lib.check(rc, "pofa_build")
        return self

    def occupied_leaves(self) -> torch.Tensor:
        return torch.nonzero(self.directory.counts > 0).reshape(-1).to(torch.int64)


def chain_indices(heads, prev, code: int) -> np.ndarray:
    """Pool indices reachable from a head, most recent first
    (fhv/storage.py:479-486); walks the device list (fhv_chain_indices)."""
    if not (isinstance(heads, torch.Tensor) and heads.is_cuda):
        raise FhvError("chain_indices: heads must be a CUDA tensor of this package")
    dev = heads.device
    h = heads if heads.dtype == torch.int32 and heads.is_contiguous() else heads.to(torch.int32).contiguous()
    p = prev if prev.dtype == torch.int32 and prev.is_contiguous() else prev.to(dev, torch.int32).contiguous()
    n = ctypes.c_int64(0)
    lib = _lib.load()
    cap = 64
    while True:
        out = torch.empty(cap, dtype=torch.int64, device=dev)
        rc = lib.fhv_chain_indices(_lib.ctx(dev), _lib.ptr(h), h.numel(), _lib.ptr(p), p.numel(), int(code), cap,
                                   _lib.ptr(out), ctypes.byref(n), _lib.stream_ptr(dev))
        if rc == _lib.FHV_BAD_ARGS:
            raise FhvError(f"chain_indices: bad key {code} or corrupt chain")
        _lib.check(rc, "chain_indices")
        if n.value <= cap:
            return out[:n.value].cpu().numpy()
        cap = int(n.value)


_chain = chain_indices


# ---------------------------------------------------------------------------
# builders (C ABI)


def _flags(alloc: str, exact_order: bool) -> int:
    if alloc not in ("ordered", "atomic"):
        raise FhvError(f"unknown alloc mode {alloc!r}")
    return (_lib.FHV_ALLOC_ATOMIC if alloc == "atomic" else 0) | (_lib.FHV_EXACT_ORDER if exact_order else 0)


def build_ppfl(scene: Scene, cfg: RasterConfig, strategy: CaptureStrategy | None = None,
               capacity: int | None = None, overalloc: float = 10.0, threads: int = 1, *,
               exact_order: bool = False, alloc: str = "ordered", device=None) -> FhvPpfl:
    """Per-pixel linked lists (fhv/storage.py:553-571); OneView only."""
    strategy = strategy or CaptureStrategy.one_view()
    if strategy.kind != "one_view":
        raise FhvError("per-pixel layout requires the single-view strategy")
    w, h = cfg.resolution
    if capacity is None:
        capacity = int(w * h * overalloc)
    plan, c = _plan_cfg(scene, strategy, cfg)
    ds = device_scene(scene, device)
    dev = ds.device
    pool = FragmentPool(capacity, dev)
    heads = torch.full((w * h,), -1, dtype=torch.int32, device=dev)
    nf = ctypes_i64()
    lib = _lib.load()
    tris, p = ds.struct(), pool.struct()
    rc = lib.fhv_build_ppfl(_lib.ctx(dev), tris, c, w, p, _lib.ptr(heads), _flags(alloc, exact_order), nf,
                            _lib.stream_ptr(dev))
    _lib.check(rc, "build_ppfl", allow=(_lib.FHV_OK, _lib.FHV_OVERFLOW))
    pool.next_free = int(nf.value)
    pool.overflowed = pool.next_free > pool.capacity
    return FhvPpfl(PixelDirectory(w, h, heads), pool, h, plan.stats(pool.next_free), scene.materials)


def build_pofl(scene: Scene, strategy: CaptureStrategy, cfg: RasterConfig, levels: int,
               capacity: int | None = None, overalloc: float = 10.0, threads: int = 1, *,
               exact_order: bool = False, alloc: str = "ordered", device=None, sync: bool = True,
               ticket: torch.Tensor | None = None) -> FhvPofl:
    """Per-octant linked lists + occupancy pyramid (fhv/storage.py:574-587).

    ``sync=False`` (once a build of the same scene / plan has run): nothing
    waits for the device -- the pool is sized by the capacity as usual,
    ``next_free`` is the last exact total, and the outcome goes to ``ticket``
    (pinned int64[4]); :meth:`FhvPofl.wait` checks it and rebuilds in place
    when the speculation (item plan, total) was wrong."""
    if levels < 1:
        raise FhvError("octree needs at least one level")
    _check_levels(levels)
    w, h = cfg.resolution
    if capacity is None:
        capacity = int(w * h * overalloc)
    plan, c = _plan_cfg(scene, strategy, cfg)
    ds = device_scene(scene, device)
    dev = ds.device
    pool = FragmentPool(capacity, dev)
    heads = torch.full((8 ** levels,), -1, dtype=torch.int32, device=dev)
    pyr = OccupancyPyramid(levels, device=dev)
    lib = _lib.load()
    tris, p = ds.struct(), pool.struct()
    guesses = ds.__dict__.setdefault("_pofl_totals", {})
    gkey = (plan.key, levels, capacity, alloc, exact_order)
    guess = guesses.get(gkey)
    if not sync and guess is not None:
        tk = ticket if ticket is not None else torch.zeros(4, dtype=torch.int64).pin_memory()
        rc = lib.fhv_build_pofl_async(_lib.ctx(dev), tris, c, levels, p, _lib.ptr(heads), _lib.ptr(pyr.data),
                                      _flags(alloc, exact_order), c_vp_of(tk), _lib.stream_ptr(dev))
        _lib.check(rc, "build_pofl")
        pool.next_free = guess
        pool.overflowed = guess > pool.capacity
        pool.in_unit_cube = True
        vol = FhvPofl(PoflDirectory(levels, heads), pyr, pool, h, plan.stats(guess), scene.materials)
        vol.pending = (tk, guess, lambda: build_pofl(scene, strategy, cfg, levels, capacity, overalloc, threads,
                                                     exact_order=exact_order, alloc=alloc, device=device))
        if not torch.cuda.is_current_stream_capturing():
            done = torch.cuda.Event()
            done.record(torch.cuda.current_stream(dev))
            vol.done = done
        return vol
    nf = ctypes_i64()
    rc = lib.fhv_build_pofl(_lib.ctx(dev), tris, c, levels, p, _lib.ptr(heads), _lib.ptr(pyr.data),
                            _flags(alloc, exact_order), nf, _lib.stream_ptr(dev))
    _lib.check(rc, "build_pofl", allow=(_lib.FHV_OK, _lib.FHV_OVERFLOW))
    pool.next_free = int(nf.value)
    guesses[gkey] = pool.next_free
    pool.overflowed = pool.next_free > pool.capacity
    pool.in_unit_cube = True
    return FhvPofl(PoflDirectory(levels, heads), pyr, pool, h, plan.stats(pool.next_free), scene.materials)


def pofa_build(scene: Scene, strategy: CaptureStrategy, cfg: RasterConfig, levels: int, threads: int = 1, *,
               exact_order: bool = True, device=None, tris=None, sync: bool = True,
               ticket: torch.Tensor | None = None) -> FhvPofa:
    """Two-pass per-octant arrays (fhv/storage.py:590-621): per-leaf histogram,
    exclusive scan (+ pyramid), exact pool, scatter into leaf ranges.
    ``exact_order`` (default, the reference's pool byte for byte): records of a
    leaf in emission order, restored by a slot-order fix-up that re-sorts only
    the leaves several warps wrote; ``exact_order=False`` keeps the paper's
    atomic in-leaf order (per-leaf multiset equal).
    ``tris``: a DeviceScene already holding this scene's triangle arrays (e.g.
    one of several buffers a pipelined caller fills asynchronously); default:
    the scene's cached upload.

    ``sync=False`` (once a build of the same scene / plan has run): nothing
    waits for the device -- the pool is sized by the last exact total and the
    outcome is written to ``ticket`` (pinned int64[4], allocated if omitted);
    call :meth:`FhvPofa.wait` (or :func:`check_ticket` after a stream sync)
    before trusting the volume on the host.  ``wait`` rebuilds synchronously
    in place when the speculation was wrong."""
    if levels < 1:
        raise FhvError("octree needs at least one level")
    if levels > 10:
        raise FhvError(f"levels {levels}: dense POFA directories beyond L=10 (8^10 leaves, 4 GiB of offsets + counts) "
                       "are not supported on the device")
    plan, c = _plan_cfg(scene, strategy, cfg)
    ds = tris if tris is not None else device_scene(scene, device)
    dev = ds.device
    n_leaf = 8 ** levels
    counts = torch.empty(n_leaf, dtype=torch.uint32, device=dev)
    offsets = torch.empty(n_leaf, dtype=torch.uint32, device=dev)
    pyr = OccupancyPyramid.uninitialized(levels, dev)  # the directory pass writes every level
    lib = _lib.load()
    total = ctypes_i64()
    cx = _lib.ctx(dev)
    st = _lib.stream_ptr(dev)
    flags = _lib.FHV_EXACT_ORDER if exact_order else 0
    # the exact pool size is data dependent: start from the last total seen for
    # this (scene, plan, levels) so count + directory + scatter run in ONE call
    # with the syncs inside the library; a miss costs a second call
    guesses = ds.__dict__.setdefault("_pofa_totals", {})
    gkey = (plan.key, levels)
    guess = guesses.get(gkey)
    if not sync and guess:
        pool = FragmentPool(guess, dev, fill_prev=False)
        tk = ticket if ticket is not None else torch.zeros(4, dtype=torch.int64).pin_memory()
        rc = lib.fhv_pofa_build_async(_lib.ctx(dev), ds.struct(), c, levels, _lib.ptr(counts), _lib.ptr(offsets),
                                      _lib.ptr(pyr.data), pool.struct(), _lib.FHV_EXACT_ORDER if exact_order else 0,
                                      c_vp_of(tk), _lib.stream_ptr(dev))
        _lib.check(rc, "pofa_build")
        pool.next_free = guess
        pool.in_unit_cube = True
        vol = FhvPofa(PofaDirectory(levels, offsets, counts), pyr, pool, int(cfg.resolution[1]), plan.stats(guess),
                      scene.materials)
        vol.pending = (tk, guess, lambda: pofa_build(scene, strategy, cfg, levels, threads, exact_order=exact_order,
                                                     device=device, tris=tris))
        if not torch.cuda.is_current_stream_capturing():
            done = torch.cuda.Event()  # after the ticket copy, on the build's own stream
            done.record(torch.cuda.current_stream(dev))
            vol.done = done
        return vol
    pool = FragmentPool(guess, dev, fill_prev=False) if guess is not None else None  # pass 2 writes every prev
    tr = ds.struct()
    rc = lib.fhv_pofa_build(cx, tr, c, levels, _lib.ptr(counts), _lib.ptr(offsets), _lib.ptr(pyr.data),
                            pool.struct() if pool is not None else None, flags, total, st)
    n = int(total.value)
    if rc == _lib.FHV_NEED_POOL:
        pool = FragmentPool(n, dev, fill_prev=False)
        rc = lib.fhv_pofa_scatter(cx, tr, c, levels, _lib.ptr(counts), _lib.ptr(offsets), pool.struct(), flags, st)
    _lib.check(rc, "pofa_build")
    guesses[gkey] = n
    if pool.capacity != n:
        pool = pool.narrow(n)
    pool.next_free = n
    pool.in_unit_cube = True
    return FhvPofa(PofaDirectory(levels, offsets, counts), pyr, pool, int(cfg.resolution[1]),
                   plan.stats(pool.next_free), scene.materials)


def c_vp_of(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


def check_ticket(vol) -> int:
    """Status of an asynchronous pofa_build (the stream must have been
    synchronised): FHV_OK, FHV_STALE (speculation wrong, outputs invalid) or
    the build's own error code."""
    tk, guess, _ = vol.pending
    if getattr(vol, "done", None) is not None:
        vol.done.synchronize()
    return ticket_status(tk, guess)


def ticket_status(ticket: torch.Tensor, guess: int) -> int:
    """fhv_ticket_check of one pinned ticket against the pool size it was built with."""
    return int(_lib.load().fhv_ticket_check(c_vp_of(ticket), int(guess)))


def _plan_cfg(scene: Scene, strategy: CaptureStrategy, cfg: RasterConfig):
    """capture_plan + its C struct, cached on the scene per (strategy, config)."""
    key = (strategy.kind, getattr(strategy, "axis", None), tuple(cfg.resolution), cfg.extent,
           np.asarray(cfg.projection).tobytes())
    cache = scene.__dict__.setdefault("_plan_cache", {})
    hit = cache.get(key)
    if hit is None:
        plan = capture_plan(scene, strategy, cfg)
        plan.key = key
        hit = cache[key] = (plan, capture_cfg(plan))
    return hit


def ctypes_i64():
    import ctypes
    return ctypes.c_int64(0)


def rebuild_pofl_as_pofa(fhv: FhvPofl) -> FhvPofa:
    """Repack a POFL into POFA (fhv/storage.py:624-652) on the device: leaf
    histogram of the f32 positions, offsets + pyramid (the POFA directory
    kernel), scatter into leaf ranges, stable in-leaf order restored by pool
    index.  Records: same bytes as the reference's lexsort repack."""
    pool = fhv.pool
    n, L, dev = pool.stored_count, fhv.levels, pool.device
    counts = torch.empty(8 ** L, dtype=torch.uint32, device=dev)
    offsets = torch.empty(8 ** L, dtype=torch.uint32, device=dev)
    pyr = OccupancyPyramid(L, device=dev)
    new = FragmentPool(n, dev, fill_prev=False)  # every prev is written (-1)
    lib = _lib.load()
    rc = lib.fhv_rebuild_pofa(_lib.ctx(dev), L, pool.struct(), n, _lib.ptr(counts), _lib.ptr(offsets),
                              _lib.ptr(pyr.data), new.struct(), _lib.stream_ptr(dev))
    _lib.check(rc, "rebuild_pofl_as_pofa")
    new.next_free = n
    new.in_unit_cube = True
    return FhvPofa(PofaDirectory(L, offsets, counts), pyr, new, fhv.capture_resolution, fhv.stats, fhv.materials)


# ---------------------------------------------------------------------------
# memory accounting (fhv/storage.py:659-719; host arithmetic)


def memory_report(layout: str, *, resolution=None, levels=None, record_size: int = RECORD_SIZE_ALIGNED,
                  capacity=None, exact_count=None, overalloc: float = 10.0, gbuffer_payload_bytes: int = 28) -> dict:
    if record_size not in (RECORD_SIZE_PACKED, RECORD_SIZE_ALIGNED):
        raise FhvError(f"record_size must be 36 or 48, got {record_size}")
    comp: dict = {}
    params: dict = {"record_size": record_size}
    if layout == "DS":
        if resolution is None:
            raise FhvError("DS report needs a resolution")
        w, h = resolution
        comp["gbuffer"] = w * h * gbuffer_payload_bytes
        params.update(gbuffer_payload_bytes=gbuffer_payload_bytes, resolution=[w, h])
    elif layout == "PPFL":
        if resolution is None:
            raise FhvError("PPFL report needs a resolution")
        w, h = resolution
        capacity = int(w * h * overalloc) if capacity is None else capacity
        comp["pixel_directory"] = 4 * w * h
        comp["fragment_pool"] = record_size * capacity
        params.update(resolution=[w, h], capacity=capacity, overalloc=overalloc)
    elif layout == "POFL":
        if levels is None:
            raise FhvError("POFL report needs levels")
        if capacity is None:
            if resolution is None:
                raise FhvError("POFL report needs a capacity or a resolution")
            capacity = int(resolution[0] * resolution[1] * overalloc)
        comp["octree_nodes"] = 4 * sum(8 ** k for k in range(levels + 1))
        comp["fragment_pool"] = record_size * capacity
        params.update(levels=levels, capacity=capacity, overalloc=overalloc)
    elif layout == "POFA":
        if levels is None or exact_count is None:
            raise FhvError("POFA report needs levels and an exact count")
        comp["octree_inner_nodes"] = 4 * sum(8 ** k for k in range(levels))
        comp["leaf_directory"] = 8 * (8 ** levels)
        comp["fragment_pool"] = record_size * exact_count
        params.update(levels=levels, exact_count=exact_count)
    else:
        raise FhvError(f"unknown layout {layout!r}")
    total = sum(comp.values())
    return {"layout": layout, "params": params, "components": comp, "total_bytes": total,
            "total_mib": total / (1024.0 * 1024.0)}


# ---------------------------------------------------------------------------
# FHV1 snapshots (fhv/storage.py:725-808), byte-exact with the reference

SNAPSHOT_MAGIC = b"FHV1"
_HEADER = struct.Struct("<4s4sIIIIQ")


def _pack_pool(pool: FragmentPool, n: int) -> torch.Tensor:
    """The first n records as packed 36-byte RECORD_DTYPE rows, on the device."""
    out = torch.empty(36 * n, dtype=torch.uint8, device=pool.device)
    rc = _lib.load().fhv_pack_records(_lib.ctx(pool.device), pool.struct(), n, _lib.ptr(out),
                                      _lib.stream_ptr(pool.device))
    _lib.check(rc, "snapshot pack")
    return out


def snapshot_bytes(fhv) -> bytes:
    """FHV1 snapshot (fhv/storage.py:725-755): header, directory, pyramid
    levels, packed records.  Assembled in device memory (records packed by a
    kernel straight from the SoA pool) and read back in ONE copy."""
    pool = fhv.pool
    count = pool.stored_count
    if fhv.layout == "PPFL":
        d = fhv.directory
        header = _HEADER.pack(SNAPSHOT_MAGIC, b"PPFL", 0, d.width, d.height, RECORD_SIZE_PACKED, count)
        planes = [d.heads]
    elif fhv.layout in ("POFL", "POFA"):
        r = fhv.capture_resolution
        header = _HEADER.pack(SNAPSHOT_MAGIC, fhv.layout.encode(), fhv.levels, r, r, RECORD_SIZE_PACKED, count)
        planes = [fhv.directory.heads] if fhv.layout == "POFL" else [fhv.directory.offsets, fhv.directory.counts]
        planes.append(fhv.pyramid.data)
    else:
        raise FhvError(f"cannot snapshot layout {fhv.layout!r}")
    planes = [t.contiguous().view(torch.uint8).reshape(-1) for t in planes] + [_pack_pool(pool, count)]
    body = torch.cat(planes) if planes else torch.empty(0, dtype=torch.uint8)
    return header + body.cpu().numpy().tobytes()


def save_snapshot(fhv, path) -> None:
    with open(path, "wb") as fh:
        fh.write(snapshot_bytes(fhv))


def load_snapshot(path, materials=None, device=None):
    blob = open(path, "rb").read()
    if len(blob) < _HEADER.size:
        raise FhvError("snapshot truncated")
    magic, layout, levels, w, h, rec, count = _HEADER.unpack_from(blob)
    if magic != SNAPSHOT_MAGIC:
        raise FhvError("bad snapshot magic")
    if rec != RECORD_SIZE_PACKED:
        raise FhvError(f"unsupported record size {rec}")
    dev = default_device(device)
    off = _HEADER.size

    def take(dtype, n):
        nonlocal off
        a = np.frombuffer(blob, dtype=dtype, count=n, offset=off).copy()
        off += a.nbytes
        return a

    def dev32(a):
        return torch.from_numpy(a.view(np.int32)).to(dev)

    def records(n):
        # validated on the host like the reference (np.frombuffer raises on a
        # short buffer), then ONE upload of the packed rows, unpacked by a kernel
        rec = take(RECORD_DTYPE, n)
        pool = FragmentPool(n, dev, fill_prev=False)
        raw = torch.from_numpy(rec.view(np.uint8).reshape(-1)).to(dev)
        rc = _lib.load().fhv_unpack_records(_lib.ctx(dev), _lib.ptr(raw), n, pool.struct(), _lib.stream_ptr(dev))
        _lib.check(rc, "snapshot unpack")
        pool.next_free = n
        return pool

    if layout == b"PPFL":
        heads = take("<i4", w * h)
        pool = records(count)
        return FhvPpfl(PixelDirectory(w, h, dev32(heads)), pool, h, materials=materials)
    if layout in (b"POFL", b"POFA"):
        if layout == b"POFL":
            heads = take("<i4", 8 ** levels)
        else:
            offs = take("<u4", 8 ** levels)
            cnts = take("<u4", 8 ** levels)
        pyr = np.concatenate([take(np.uint8, 8 ** k) for k in range(levels)])
        pool = records(count)
        pyramid = OccupancyPyramid(levels, torch.from_numpy(pyr).to(dev))
        if layout == b"POFL":
            return FhvPofl(PoflDirectory(levels, dev32(heads)), pyramid, pool, h, materials=materials)
        return FhvPofa(PofaDirectory(levels, dev32(offs).view(torch.uint32), dev32(cnts).view(torch.uint32)),
                       pyramid, pool, h, materials=materials)
    raise FhvError(f"unknown snapshot layout {layout!r}")


# ---------------------------------------------------------------------------
# per-fragment / per-batch insertion (fhv/storage.py:331-476): the sink
# objects capture_pass can feed and the single-fragment inserts.  Records are
# written into the device pool; chaining, cursor assignment and occupancy run
# in the operator kernels (kernels.linked_insert / pofa_scatter, set_paths).
# The bulk builders above never go through these.


def _dev_rows(a, dev, dtype) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).astype(
        {torch.float32: np.float32, torch.int64: np.int64}[dtype]))).to(dev)


def _store_split(pool: FragmentPool, n: int) -> tuple:
    start = pool.alloc_block(n)
    return start, min(n, max(0, pool.capacity - start))


def _write_records(pool: FragmentPool, dest, batch, stored: int) -> np.ndarray:
    """Write batch[:stored] at pool slots ``dest`` (a slice or index tensor); returns f32 positions (host)."""
    dev = pool.device
    pos32 = np.asarray(batch.world_position[:stored], dtype=np.float64).astype(np.float32).reshape(-1, 3)
    nrm32 = np.asarray(batch.world_normal[:stored], dtype=np.float64).astype(np.float32).reshape(-1, 3)
    pool.position[dest] = torch.from_numpy(pos32).to(dev)
    pool.normal[dest] = torch.from_numpy(nrm32).to(dev)
    pool.material_id.view(torch.int32)[dest] = int(np.uint32(batch.material_id).view(np.int32))
    pool.object_id.view(torch.int32)[dest] = int(np.uint32(batch.object_id).view(np.int32))
    return pos32


class PpflSink:
    """capture_pass sink into a per-pixel linked-list layout (fhv/storage.py:356-373)."""

    def __init__(self, directory: PixelDirectory, pool: FragmentPool):
        self.directory = directory
        self.pool = pool
        self._lock = threading.Lock()

    def __call__(self, batch) -> None:
        from . import kernels
        with self._lock:
            start, stored = _store_split(self.pool, len(batch))
            if stored == 0:
                return
            _write_records(self.pool, slice(start, start + stored), batch, stored)
            keys = (np.asarray(batch.raster_y[:stored], dtype=np.int64) * self.directory.width
                    + np.asarray(batch.raster_x[:stored], dtype=np.int64))
            kernels.linked_insert(keys, self.directory.heads, self.pool.prev_index, start)


class PoflSink:
    """capture_pass sink into a per-octant linked-list layout (fhv/storage.py:376-395)."""

    def __init__(self, directory: PoflDirectory, pyramid: OccupancyPyramid, pool: FragmentPool):
        self.directory = directory
        self.pyramid = pyramid
        self.pool = pool
        self._lock = threading.Lock()

    def __call__(self, batch) -> None:
        from . import kernels
        with self._lock:
            start, stored = _store_split(self.pool, len(batch))
            if stored == 0:
                return
            pos32 = _write_records(self.pool, slice(start, start + stored), batch, stored)
            codes = np.atleast_1d(cell_code(pos32.astype(np.float64), self.directory.levels))
            kernels.linked_insert(codes, self.directory.heads, self.pool.prev_index, start)
            self.pyramid.set_paths(codes)


class CountingSink:
    """First POFA pass: fragments per leaf (fhv/storage.py:398-410); ``counts``
    is an int64 device tensor of 8^levels."""

    def __init__(self, levels: int, device=None):
        self.levels = levels
        self.counts = torch.zeros(8 ** levels, dtype=torch.int64, device=default_device(device))
        self._lock = threading.Lock()

    def __call__(self, batch) -> None:
        pos32 = np.asarray(batch.world_position, dtype=np.float64).astype(np.float32).reshape(-1, 3)
        codes = np.atleast_1d(cell_code(pos32.astype(np.float64), self.levels))
        c = torch.from_numpy(np.ascontiguousarray(codes, dtype=np.int64)).to(self.counts.device)
        with self._lock:
            self.counts.index_add_(0, c, torch.ones_like(c))


class PofaWriteSink:
    """Second POFA pass: scatter fragments to their leaf ranges (fhv/storage.py:413-439)."""

    def __init__(self, directory: PofaDirectory, pool: FragmentPool):
        self.directory = directory
        self.pool = pool
        self.cursors = torch.zeros(directory.counts.numel(), dtype=torch.int32,
                                   device=directory.counts.device).view(torch.uint32)
        self._lock = threading.Lock()

    def __call__(self, batch) -> None:
        from . import kernels
        with self._lock:
            n = len(batch)
            pos32 = np.asarray(batch.world_position, dtype=np.float64).astype(np.float32).reshape(-1, 3)
            codes = np.atleast_1d(cell_code(pos32.astype(np.float64), self.directory.levels))
            dest = torch.empty(n, dtype=torch.int64, device=self.pool.device)
            bad = kernels.pofa_scatter(codes, self.directory.offsets, self.directory.counts, self.cursors, dest)
            if bad >= 0:
                raise PofaBuildError(f"octant {int(codes[bad])} received more fragments than counted")
            self.pool.alloc_block(n)
            _write_records(self.pool, dest, batch, n)
            self.pool.prev_index[dest] = -1


def ppfl_insert(directory: PixelDirectory, pool: FragmentPool, frag) -> int | None:
    """Insert one fragment; its pool index, or None on overflow (fhv/storage.py:442-458)."""
    from . import kernels
    x, y = frag.raster_xy
    if not (0 <= x < directory.width and 0 <= y < directory.height):
        raise FhvError(f"raster position {frag.raster_xy} out of range")
    idx = pool.alloc_block(1)
    if idx >= pool.capacity:
        return None
    _write_records(pool, slice(idx, idx + 1), _One(frag), 1)
    kernels.linked_insert(np.array([y * directory.width + x], dtype=np.int64), directory.heads, pool.prev_index, idx)
    return idx


def pofl_insert(directory: PoflDirectory, pyramid: OccupancyPyramid, pool: FragmentPool, frag) -> int | None:
    """Insert one fragment keyed by its Morton leaf; updates occupancy (fhv/storage.py:461-476)."""
    from . import kernels
    idx = pool.alloc_block(1)
    if idx >= pool.capacity:
        return None
    pos32 = _write_records(pool, slice(idx, idx + 1), _One(frag), 1)
    code = int(np.atleast_1d(cell_code(pos32[0].astype(np.float64), directory.levels))[0])
    kernels.linked_insert(np.array([code], dtype=np.int64), directory.heads, pool.prev_index, idx)
    pyramid.set_paths(np.array([code], dtype=np.int64))
    return idx


class _One:
    """An EmittedFragment seen as a one-row batch."""

    def __init__(self, frag):
        self.world_position = np.asarray(frag.world_position, dtype=np.float64).reshape(1, 3)
        self.world_normal = np.asarray(frag.world_normal, dtype=np.float64).reshape(1, 3)
        self.material_id = frag.material_id
        self.object_id = frag.object_id
