"""Multi-GPU partition of the hot path by Morton range.

The reference is single-process (no distribution at all, SURVEY.md section 2
row 13); this module is the B200 build's scale-out of its POFA capture
(``pofa_build``, fhv/storage.py:590-621) and splat reconstruction
(``splat_render``, fhv/render.py:249-320) across the GPUs of one box:

* **Capture.**  Rank r owns the contiguous leaf range ``[lo_r, hi_r)`` of the
  Morton order (whole directory tiles of 8^5 leaves).  It rasterises only the
  triangles whose f64 AABB meets its range's world-space cover (binning on the
  device), keeps only fragments of its own leaves, and builds its slice of the
  directory.  The single exchange is one ``all_gather`` of a fragment total
  per rank: ``base_r`` = sum of the lower ranks' totals turns local offsets
  into global ones.  Leaf order inside the Morton range equals the global
  order restricted to it, so the concatenation of the ranks' pools and
  directory slices IS the 1-GPU ``pofa_build`` (bit-identical with
  ``exact_order=True``; the tests check it).
* **Splat.**  Each rank z-tests its own fragments into a full-frame int64
  depth-key buffer; ``all_reduce(MIN)`` composites the ranks by depth; the
  tie-break pass finds each pixel's lowest global pool index among the
  fragments at the global depth, ``all_reduce(MIN)``; each rank shades the
  pixels whose winner it owns (-0.0 elsewhere, the exact neutral element of
  addition) and ``all_reduce(SUM)`` assembles the frame.  Identical to
  ``splat_render`` over the whole pool.

``Comm`` is the exchange: ``TorchComm`` (torch.distributed, NCCL over
NVLink on the box, gloo on CPU) or ``ThreadComm`` (N ranks as threads of one
process sharing one GPU -- a loopback used by the tests).
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import DeviceShading, capture_cfg, device_scene, host_f64
from .lights import ImageBuffer
from .raster import CaptureStrategy, RasterConfig, capture_plan
from .raycast import primary_rays
from .scene import Camera, SceneError
from .storage import FhvError, FragmentPool, OccupancyPyramid, PofaDirectory, _check_levels, morton_decode

__all__ = ["Comm", "FhvPofaShard", "ThreadComm", "TorchComm", "fragment_weights", "pofa_build_shard",
           "range_boxes", "render_raycast_shard", "shard_ranges", "splat_render_shard", "tile_leaves", "PeerFrame"]

MAX_BOXES = 64
BIN_MARGIN = 1e-5  # world units; fragments lie within 1 f32 ulp of the triangle's AABB


# ---------------------------------------------------------------------------
# partition


def tile_leaves(levels: int) -> int:
    """Leaves per directory tile = the granularity of a shard range."""
    if levels >= 5:
        return 8 ** 5
    if levels == 4:
        return 8 ** 4
    raise FhvError("sharded capture needs levels >= 4")


def shard_ranges(levels: int, world: int, weights: np.ndarray | None = None) -> list:
    """Contiguous Morton ranges [lo, hi), one per rank, cut at tile bounds.
    ``weights`` (one per tile, e.g. :func:`fragment_weights`) balances the
    expected fragments per rank; otherwise the tiles are split evenly."""
    _check_levels(levels)
    tl = tile_leaves(levels)
    n_tiles = 8 ** levels // tl
    if world < 1 or world > n_tiles:
        raise FhvError(f"cannot split {n_tiles} directory tiles across {world} ranks")
    if weights is None:
        cuts = [round(r * n_tiles / world) for r in range(world + 1)]
    else:
        w = np.asarray(weights, dtype=np.float64)
        if w.shape != (n_tiles,):
            raise FhvError("weights must have one entry per directory tile")
        cum = np.concatenate(([0.0], np.cumsum(w)))
        total = cum[-1]
        cuts = [0]
        for r in range(1, world):
            c = int(np.searchsorted(cum, total * r / world, side="left"))
            c = min(max(c, cuts[-1] + 1), n_tiles - (world - r))  # every rank keeps >= 1 tile
            cuts.append(c)
        cuts.append(n_tiles)
    return [(cuts[r] * tl, cuts[r + 1] * tl) for r in range(world)]


def range_boxes(lo: int, hi: int, levels: int) -> np.ndarray:
    """World-space cover of leaves [lo, hi): the range split into aligned
    Morton blocks (each an octree node, i.e. a cube).  Falls back to the
    blocks' bounding box beyond MAX_BOXES blocks."""
    boxes = []
    while lo < hi:
        k = 0
        while k < levels and lo % (8 ** (k + 1)) == 0 and lo + 8 ** (k + 1) <= hi:
            k += 1
        lvl = levels - k
        x, y, z = morton_decode(lo >> (3 * k), lvl) if lvl > 0 else (0, 0, 0)
        size = 1.0 / (1 << lvl)
        boxes.append((x * size, y * size, z * size, (x + 1) * size, (y + 1) * size, (z + 1) * size))
        lo += 8 ** k
    b = np.asarray(boxes, dtype=np.float64).reshape(-1, 6)
    if len(b) > MAX_BOXES:
        b = np.concatenate((b[:, :3].min(axis=0), b[:, 3:].max(axis=0)))[None, :]
    return b


def fragment_weights(scene, strategy: CaptureStrategy, cfg: RasterConfig, levels: int) -> np.ndarray:
    """Expected fragments per directory tile, for balanced ranges: each
    triangle's area / pitch^2 (x3 for the three-axis strategies) binned by its
    centroid.  Host NumPy, cached on the scene (planning, not the hot path)."""
    key = ("fragment_weights", strategy.kind, cfg.resolution, cfg.extent, levels)
    cache = scene.__dict__.setdefault("_shard_cache", {})
    if key in cache:
        return cache[key]
    tl = tile_leaves(levels)
    tlev = levels - int(round(np.log(tl) / np.log(8)))  # octree level of a tile
    pos = np.asarray(scene.positions, dtype=np.float64)
    cen = np.clip(pos.mean(axis=1), 0.0, 1.0)
    side = 1 << tlev
    idx = np.clip(np.floor(cen * side).astype(np.int64), 0, side - 1)
    from .storage import morton_encode
    code = morton_encode(idx[:, 0], idx[:, 1], idx[:, 2], tlev) if tlev > 0 else np.zeros(len(pos), np.int64)
    e1, e2 = pos[:, 1] - pos[:, 0], pos[:, 2] - pos[:, 0]
    area = 0.5 * np.linalg.norm(np.cross(e1, e2), axis=1)
    pitch = cfg.extent / cfg.resolution[1]
    w = area / (pitch * pitch) * (3.0 if strategy.kind in ("three_separate", "three_way_geometry") else 1.0)
    out = np.bincount(code, weights=w + 1.0, minlength=8 ** tlev).astype(np.float64)
    cache[key] = out
    return out


# ---------------------------------------------------------------------------
# exchange


class Comm:
    rank: int = 0
    world: int = 1
    device: torch.device | None = None

    def all_gather_int(self, v: int) -> list:
        raise NotImplementedError

    def all_reduce_(self, t: torch.Tensor, op: str) -> torch.Tensor:
        raise NotImplementedError

    def barrier(self) -> None:
        """Every rank's device work issued so far is complete on return."""
        raise NotImplementedError

    def all_gather_tensor(self, t: torch.Tensor) -> list:
        """Every rank's tensor (same shape / dtype), in rank order."""
        raise NotImplementedError

    def peer_alloc(self, shapes_dtypes: list, device) -> tuple:
        """Peer-visible device buffers: (local tensors, per-rank lists of the
        buffers' device pointers as mapped in THIS process)."""
        raise NotImplementedError


class TorchComm(Comm):
    """torch.distributed over the default (or given) process group.  NCCL
    operates on the CUDA tensors directly (NVLink / NVSwitch); gloo on CPU
    copies."""

    _OPS = {"min": "MIN", "max": "MAX", "sum": "SUM"}

    def __init__(self, group=None, device: torch.device | None = None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self.device = device

    def _dev(self):
        return self.device if self.backend == "nccl" else torch.device("cpu")

    def all_gather_int(self, v: int) -> list:
        t = torch.tensor([int(v)], dtype=torch.int64, device=self._dev())
        out = torch.empty(self.world, dtype=torch.int64, device=self._dev())
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return [int(x) for x in out.cpu().tolist()]

    def all_reduce_(self, t: torch.Tensor, op: str) -> torch.Tensor:
        rop = getattr(self.dist.ReduceOp, self._OPS[op])
        if self.backend != "nccl" and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, op=rop, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, op=rop, group=self.group)
        return t

    def barrier(self) -> None:
        if self.device is not None:
            torch.cuda.synchronize(self.device)
        self.dist.barrier(group=self.group)

    def all_gather_tensor(self, t: torch.Tensor) -> list:
        src = t.contiguous() if self.backend == "nccl" or not t.is_cuda else t.cpu()
        out = torch.empty((self.world,) + tuple(src.shape), dtype=src.dtype, device=src.device)
        self.dist.all_gather_into_tensor(out, src, group=self.group)
        return [o.to(t.device) for o in out]

    def peer_alloc(self, shapes_dtypes: list, device) -> tuple:
        # NVLink peer mappings through torch's symmetric memory (one buffer per
        # tensor, rendezvous over this group): buffer_ptrs[r] = rank r's buffer
        # in this process's address space
        import torch.distributed._symmetric_memory as symm_mem
        group = self.group if self.group is not None else self.dist.group.WORLD
        tensors, ptrs = [], [[] for _ in range(self.world)]
        for shape, dtype in shapes_dtypes:
            t = symm_mem.empty(shape, dtype=dtype, device=device)
            hdl = symm_mem.rendezvous(t, group.group_name)
            tensors.append(t)
            for r in range(self.world):
                ptrs[r].append(int(hdl.buffer_ptrs[r]))
        return tensors, ptrs


class _ThreadHub:
    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world


class ThreadComm(Comm):
    """``world`` ranks as host threads of one process (loopback on one GPU).
    Every rank reduces the published tensors in rank order, so all ranks get
    bitwise the same result."""

    def __init__(self, hub: _ThreadHub, rank: int, device: torch.device | None = None):
        self.hub, self.rank, self.world, self.device = hub, rank, hub.world, device

    @staticmethod
    def group(world: int, device: torch.device | None = None) -> list:
        hub = _ThreadHub(world)
        return [ThreadComm(hub, r, device) for r in range(world)]

    def _exchange(self, v):
        h = self.hub
        h.slots[self.rank] = v
        h.barrier.wait()
        got = list(h.slots)
        h.barrier.wait()
        return got

    def all_gather_int(self, v: int) -> list:
        return [int(x) for x in self._exchange(int(v))]

    def barrier(self) -> None:
        torch.cuda.synchronize(self.device)
        self.hub.barrier.wait()

    def all_gather_tensor(self, t: torch.Tensor) -> list:
        if t.is_cuda:
            torch.cuda.synchronize(t.device)
        parts = self._exchange(t)
        got = [p.clone() for p in parts]
        if t.is_cuda:
            torch.cuda.synchronize(t.device)
        self._exchange(None)  # every rank has copied every part before any rank reuses its own
        return got

    def peer_alloc(self, shapes_dtypes: list, device) -> tuple:
        # one process, one device: every rank's pointers are directly usable
        tensors = [torch.empty(shape, dtype=dtype, device=device) for shape, dtype in shapes_dtypes]
        mine = [t.data_ptr() for t in tensors]
        return tensors, [list(p) for p in self._exchange(mine)]

    def all_reduce_(self, t: torch.Tensor, op: str) -> torch.Tensor:
        if t.is_cuda:
            torch.cuda.synchronize(t.device)
        parts = self._exchange(t)
        fn = {"min": torch.minimum, "max": torch.maximum, "sum": torch.add}[op]
        acc = parts[0].clone()
        for p in parts[1:]:
            acc = fn(acc, p)
        if t.is_cuda:
            torch.cuda.synchronize(t.device)
        self._exchange(None)  # every rank has read every part before any rank overwrites its own
        t.copy_(acc)
        return t


# ---------------------------------------------------------------------------
# sharded capture


@dataclass
class FhvPofaShard:
    """One rank's slice of a POFA volume: leaves [cell_lo, cell_hi), pool
    records with global indices [base, base + pool.capacity)."""
    directory: PofaDirectory   # counts / offsets of the owned leaves (offsets are global)
    pyramid: OccupancyPyramid  # this shard's occupancy (see gather_pyramid)
    pool: FragmentPool
    capture_resolution: int
    cell_lo: int
    cell_hi: int
    base: int
    total: int
    rank: int
    world: int
    stats: object = None
    materials: list | None = None
    layout = "POFA"

    pending = None  # (ticket, guessed local total, collective synchronous rebuild) of a sync=False build
    done = None     # CUDA event after the asynchronous build's ticket copy

    @property
    def levels(self) -> int:
        return self.directory.levels

    def wait(self, comm: Comm) -> "FhvPofaShard":
        """Finish a speculative ``pofa_build_shard(sync=False)`` on EVERY
        rank (collective): each rank checks its ticket, the statuses are
        gathered, and if any rank's total missed its guess all ranks rebuild
        synchronously (the bases of the ranks above it were wrong too); any
        other error is raised."""
        if self.pending is None:
            comm.all_gather_int(_lib.FHV_OK)  # stay collective with ranks that do wait
            return self
        tk, guess, rebuild = self.pending
        if self.done is not None:
            self.done.synchronize()
        else:
            torch.cuda.current_stream(self.pool.device).synchronize()
        from .storage import ticket_status
        rc = ticket_status(tk, guess)
        self.pending = None
        codes = comm.all_gather_int(rc)
        bad = [c for c in codes if c not in (_lib.FHV_OK, _lib.FHV_STALE)]
        if bad:
            _lib.check(rc if rc != _lib.FHV_OK and rc != _lib.FHV_STALE else bad[0], "pofa_build_shard")
        if any(c == _lib.FHV_STALE for c in codes):
            fresh = rebuild()
            for f in ("directory", "pyramid", "pool", "base", "total", "stats"):
                setattr(self, f, getattr(fresh, f))
        return self

    def gather_pyramid(self, comm: Comm) -> OccupancyPyramid:
        """The global occupancy pyramid: MAX over ranks is exact at and below
        the tile level (each node inside one rank's range); the few levels
        above are recomputed."""
        data = self.pyramid.data.clone()
        comm.all_reduce_(data, "max")
        L = self.levels
        k_tile = L - int(round(np.log(tile_leaves(L)) / np.log(8)))
        off = [((1 << (3 * k)) - 1) // 7 for k in range(L + 1)]
        bit = (1 << torch.arange(8, device=data.device, dtype=torch.int32))
        for k in range(k_tile - 1, -1, -1):
            below = data[off[k + 1]:off[k + 2]].to(torch.int32).reshape(-1, 8)
            data[off[k]:off[k + 1]] = ((below != 0).to(torch.int32) * bit).sum(dim=1).to(torch.uint8)
        return OccupancyPyramid(L, data)


def _shard_struct(lo: int, hi: int, levels: int) -> _lib.Shard:
    sh = _lib.Shard()
    sh.cell_lo, sh.cell_hi = lo, hi
    full = lo == 0 and hi == 8 ** levels
    boxes = np.zeros((0, 6)) if full else range_boxes(lo, hi, levels)
    sh.n_boxes = len(boxes)
    sh.margin = BIN_MARGIN
    for i, b in enumerate(boxes):
        for k in range(6):
            sh.boxes[i][k] = float(b[k])
    return sh


def pofa_build_shard(scene, strategy: CaptureStrategy, cfg: RasterConfig, levels: int, comm: Comm,
                     ranges: list | None = None, balance: bool = True, exact_order: bool = True,
                     device=None, tris=None, sync: bool = True, ticket: torch.Tensor | None = None) -> FhvPofaShard:
    """This rank's share of ``pofa_build(scene, strategy, cfg, levels)``.

    ``sync=False`` (after a synchronous build of the same scene, ranges and
    rank layout): no host wait and no collective -- every rank's total is
    taken from that build (base, pool size), the triangle binning is reused
    and the outcome goes to ``ticket``; :meth:`FhvPofaShard.wait` (collective)
    checks all ranks' tickets and rebuilds if any speculation missed."""
    if levels < 4:
        raise FhvError("sharded capture needs levels >= 4")
    if levels > 11:
        raise FhvError(f"levels {levels}: dense POFA directories beyond L=11 exceed device memory")
    if ranges is None:
        w = fragment_weights(scene, strategy, cfg, levels) if balance else None
        ranges = shard_ranges(levels, comm.world, w)
    lo, hi = ranges[comm.rank]
    plan = capture_plan(scene, strategy, cfg)
    ds = tris if tris is not None else device_scene(scene, device)
    dev = ds.device
    n_local = hi - lo
    counts = torch.empty(n_local, dtype=torch.uint32, device=dev)
    offsets = torch.empty(n_local, dtype=torch.uint32, device=dev)
    pyr = OccupancyPyramid(levels, device=dev)  # zeros: only this shard's occupancy is written
    lib = _lib.load()
    tris, c = ds.struct(), capture_cfg(plan)
    sh = _shard_struct(lo, hi, levels)
    cx, st = _lib.ctx(dev), _lib.stream_ptr(dev)
    cache = ds.__dict__.setdefault("_shard_totals", {})
    ckey = (tuple(cfg.resolution), np.asarray(cfg.projection).tobytes(), strategy.kind,
            getattr(strategy, "axis", None), levels, tuple(tuple(r) for r in ranges), comm.rank, comm.world,
            bool(exact_order))
    totals = cache.get(ckey)
    if not sync and totals is not None:
        base, total, guess = sum(totals[:comm.rank]), sum(totals), totals[comm.rank]
        pool = FragmentPool(guess, dev, fill_prev=False)
        tk = ticket if ticket is not None else torch.zeros(4, dtype=torch.int64).pin_memory()
        rc = lib.fhv_pofa_shard_build_async(cx, tris, c, levels, sh, _lib.ptr(counts), _lib.ptr(offsets),
                                            _lib.ptr(pyr.data), base, pool.struct(),
                                            _lib.FHV_EXACT_ORDER if exact_order else 0, ctypes.c_void_p(tk.data_ptr()),
                                            st)
        _lib.check(rc, "pofa_build_shard")
        pool.next_free = guess
        vol = FhvPofaShard(PofaDirectory(levels, offsets, counts), pyr, pool, int(cfg.resolution[1]), lo, hi, base,
                           total, comm.rank, comm.world, plan.stats(total), scene.materials)
        vol.pending = (tk, guess, lambda: pofa_build_shard(scene, strategy, cfg, levels, comm, ranges, balance,
                                                           exact_order, device, ds))
        if not torch.cuda.is_current_stream_capturing():
            done = torch.cuda.Event()
            done.record(torch.cuda.current_stream(dev))
            vol.done = done
        return vol
    local = ctypes.c_int64(0)
    rc = lib.fhv_pofa_shard_count(cx, tris, c, levels, sh, _lib.ptr(counts), local, st)
    _lib.check(rc, "pofa_build_shard pass 1")
    totals = comm.all_gather_int(local.value)
    cache[ckey] = list(totals)
    base, total = sum(totals[:comm.rank]), sum(totals)
    if total >= 1 << 32:
        raise FhvError("fragment count exceeds the 32-bit offset range")
    rc = lib.fhv_pofa_shard_directory(cx, levels, sh, _lib.ptr(counts), _lib.ptr(offsets), _lib.ptr(pyr.data), base,
                                      st)
    _lib.check(rc, "pofa_build_shard directory")
    pool = FragmentPool(int(local.value), dev, fill_prev=False)
    rc = lib.fhv_pofa_shard_scatter(cx, tris, c, levels, sh, _lib.ptr(counts), _lib.ptr(offsets), base, pool.struct(),
                                    _lib.FHV_EXACT_ORDER if exact_order else 0, st)
    _lib.check(rc, "pofa_build_shard pass 2")
    pool.next_free = pool.capacity
    return FhvPofaShard(PofaDirectory(levels, offsets, counts), pyr, pool, int(cfg.resolution[1]), lo, hi, base, total,
                        comm.rank, comm.world, plan.stats(total), scene.materials)


# ---------------------------------------------------------------------------
# sharded splat


class SplatBuffers:
    """Per-view int64 key / winner buffers (reusable across frames)."""

    def __init__(self, width: int, height: int, device):
        self.keys = torch.empty(width * height, dtype=torch.int64, device=device)
        self.winners = torch.empty(width * height, dtype=torch.int64, device=device)


class PeerFrame:
    """Peer-visible splat buffers of one rank for a W x H view (reusable
    across frames): its row slab of depth keys and winners (rank q owns rows
    [q H / N, (q+1) H / N)) and its full-frame rgba / depth, plus the table
    of every rank's buffers as mapped in this process (fhv_peer_t)."""

    def __init__(self, width: int, height: int, comm: Comm, device):
        N, q = comm.world, comm.rank
        if N > _lib.FHV_MAX_PEERS or height < N:
            raise FhvError(f"peer splat supports up to {_lib.FHV_MAX_PEERS} ranks and height >= ranks")
        rows = (q + 1) * height // N - q * height // N
        t, ptrs = comm.peer_alloc([((rows * width,), torch.int64), ((rows * width,), torch.int64),
                                   ((height, width, 4), torch.float64), ((height, width), torch.float64)], device)
        self.keys, self.winners, self.rgba, self.depth = t
        self.width, self.height, self.comm = width, height, comm
        st = _lib.Peer()
        st.nranks, st.width, st.height = N, width, height
        for r in range(N):
            st.keys[r], st.winners[r], st.rgba[r], st.depth[r] = ptrs[r]
        self.struct = st
        self._probe(comm, device)

    def _probe(self, comm: Comm, device) -> None:
        """Each rank stamps its slab, every rank reads all stamps back through
        its peer mappings: raises if a mapping does not reach its buffer."""
        N = comm.world
        self.winners[0] = 1000 + comm.rank
        comm.barrier()
        out = torch.zeros(N, dtype=torch.int64, device=device)
        lib = _lib.load()
        cam = np.zeros(22)
        cam[13], cam[14] = self.width, self.height
        rc = lib.fhv_splat_peer(_lib.ctx(device), 4, 0, None, None, None, cam.ctypes.data, 1.0, None, None,
                                self.struct, comm.rank, 0, ctypes.c_void_p(out.data_ptr()), _lib.stream_ptr(device))
        _lib.check(rc, "peer probe")
        got = out.cpu().tolist()
        comm.barrier()
        if got != [1000 + r for r in range(N)]:
            raise FhvError(f"peer mappings do not reach the peers' buffers: {got}")


def _splat_peer(vol, camera, splat_radius_world, comm, background, out, shading, peer):
    """Peer-memory composite (fhv_splat_peer): RED.MIN into the owners' row
    slabs, winner candidates likewise, then each rank shades the winners it
    owns straight into every rank's frame; four phases separated by barriers."""
    pool = vol.pool
    dev = pool.device
    w, h = camera.resolution
    if peer is None or (peer.width, peer.height) != (w, h):
        peer = PeerFrame(w, h, comm, dev)
    n = pool.stored_count
    cam = host_f64(camera.scalars())
    bg = host_f64(background)
    lib = _lib.load()
    cx, st = _lib.ctx(dev), _lib.stream_ptr(dev)
    r = float(splat_radius_world)
    args = (n, _lib.ptr(pool.position), _lib.ptr(pool.normal), _lib.ptr(pool.material_id), cam.ctypes.data, r,
            shading.struct(), bg.ctypes.data, peer.struct, comm.rank, vol.base)
    _lib.check(lib.fhv_splat_peer(cx, 0, *args, None, st), "splat peer fill")
    comm.barrier()
    fp = (ctypes.c_int64 * 2)()
    _lib.check(lib.fhv_splat_peer(cx, 1, *args, fp, st), "splat peer keys")
    ext = torch.tensor([fp[0], fp[1]], dtype=torch.int64, device=dev)
    comm.all_reduce_(ext, "max")
    kx, ky = (int(v) for v in ext.cpu().tolist())
    if kx * ky > 4096:
        _lib.check(_lib.FHV_SPLAT_BIG, "splat_render_shard")
    comm.barrier()
    _lib.check(lib.fhv_splat_peer(cx, 2, *args, None, st), "splat peer winners")
    comm.barrier()
    _lib.check(lib.fhv_splat_peer(cx, 3, *args, None, st), "splat peer resolve")
    comm.barrier()
    out.pixels.copy_(peer.rgba)
    out.depth.copy_(peer.depth)
    return out


def splat_render_shard(vol: FhvPofaShard, camera: Camera, lights, splat_radius_world: float, materials, comm: Comm,
                       background=(0.0, 0.0, 0.0, 0.0), *, out: ImageBuffer | None = None,
                       shading: DeviceShading | None = None, buffers: SplatBuffers | None = None,
                       composite: str = "allreduce", peer: PeerFrame | None = None) -> ImageBuffer:
    """``splat_render`` of the union of all ranks' pools; every rank returns
    the full frame.  ``composite="allreduce"``: key / winner / pixel planes
    combined with collective all-reduces (NCCL); ``"peer"``: written straight
    into the owner's / every rank's buffers over peer memory (fhv_splat_peer,
    ``peer`` = a reusable PeerFrame)."""
    if splat_radius_world <= 0.0:
        raise SceneError("splat radius must be > 0")
    if composite not in ("allreduce", "peer"):
        raise FhvError(f"unknown composite {composite!r}")
    pool = vol.pool
    dev = pool.device
    w, h = camera.resolution
    if out is None:
        out = ImageBuffer(w, h, torch.empty((h, w, 4), dtype=torch.float64, device=dev),
                          torch.empty((h, w), dtype=torch.float64, device=dev))
    if shading is None:
        shading = DeviceShading(materials, lights, dev)
    if composite == "peer":
        return _splat_peer(vol, camera, splat_radius_world, comm, background, out, shading, peer)
    if buffers is None:
        buffers = SplatBuffers(w, h, dev)
    n = pool.stored_count
    cam = host_f64(camera.scalars())
    bg = host_f64(background)
    lib = _lib.load()
    cx, st = _lib.ctx(dev), _lib.stream_ptr(dev)
    r = float(splat_radius_world)
    fp = (ctypes.c_int64 * 2)()
    rc = lib.fhv_splat_shard_keys(cx, n, _lib.ptr(pool.position), cam.ctypes.data, r, _lib.ptr(buffers.keys), fp, st)
    _lib.check(rc, "splat_render_shard keys")
    ext = torch.tensor([fp[0], fp[1]], dtype=torch.int64, device=dev)
    comm.all_reduce_(ext, "max")
    kx, ky = (int(v) for v in ext.cpu().tolist())
    if kx * ky > 4096:
        _lib.check(_lib.FHV_SPLAT_BIG, "splat_render_shard")
    comm.all_reduce_(buffers.keys, "min")
    rc = lib.fhv_splat_shard_winners(cx, n, _lib.ptr(pool.position), cam.ctypes.data, r, _lib.ptr(buffers.keys),
                                     vol.base, _lib.ptr(buffers.winners), st)
    _lib.check(rc, "splat_render_shard winners")
    comm.all_reduce_(buffers.winners, "min")
    rc = lib.fhv_splat_shard_resolve(cx, n, _lib.ptr(pool.position), _lib.ptr(pool.normal), _lib.ptr(pool.material_id),
                                     cam.ctypes.data, r, shading.struct(), _lib.ptr(buffers.keys),
                                     _lib.ptr(buffers.winners), vol.base, 1 if comm.rank == 0 else 0, bg.ctypes.data,
                                     _lib.ptr(out.pixels), _lib.ptr(out.depth), st)
    _lib.check(rc, "splat_render_shard resolve")
    comm.all_reduce_(out.pixels, "sum")
    comm.all_reduce_(out.depth, "sum")
    return out


# ---------------------------------------------------------------------------
# sharded ray cast ("opaque: min-t reduction; R/T: each rank
# composites its subtree's segment into a partial (C, A); partials composited
# in per-ray entry order")


def region_box(lo: int, hi: int, levels: int):
    """The world box of leaves [lo, hi) when the range is one axis-aligned box
    (a union of whole sibling octree nodes forming a slab / quadrant / node:
    the even partitions of the top-level octants for N = 1, 2, 4, 8), else None."""
    b = range_boxes(lo, hi, levels)
    lo3, hi3 = b[:, :3].min(axis=0), b[:, 3:].max(axis=0)
    vol = float(np.prod(hi3 - lo3))
    if abs(vol - float(np.sum(np.prod(b[:, 3:] - b[:, :3], axis=1)))) > 1e-12 * max(vol, 1e-300):
        return None
    return lo3, hi3


def local_volume(vol: FhvPofaShard):
    """This rank's shard as a stand-alone POFA volume for the ray cast:
    full-size directory (zero counts outside the owned range, offsets local
    to the shard's pool) and the pyramid of the shard's own occupancy."""
    from .storage import FhvPofa
    L = vol.levels
    dev = vol.pool.device
    n = 8 ** L
    counts = torch.zeros(n, dtype=torch.uint32, device=dev)
    offsets = torch.zeros(n, dtype=torch.uint32, device=dev)
    counts[vol.cell_lo:vol.cell_hi] = vol.directory.counts
    offsets[vol.cell_lo:vol.cell_hi] = (vol.directory.offsets.to(torch.int64) - vol.base).to(torch.uint32)
    data = vol.pyramid.data.clone()
    k_tile = L - int(round(np.log(tile_leaves(L)) / np.log(8)))
    off = [((1 << (3 * k)) - 1) // 7 for k in range(L + 1)]
    bit = (1 << torch.arange(8, device=dev, dtype=torch.int32))
    for k in range(k_tile - 1, -1, -1):  # the levels above the tiles, from this shard's occupancy alone
        below = data[off[k + 1]:off[k + 2]].to(torch.int32).reshape(-1, 8)
        data[off[k]:off[k + 1]] = ((below != 0).to(torch.int32) * bit).sum(dim=1).to(torch.uint8)
    pool = vol.pool
    return FhvPofa(PofaDirectory(L, offsets, counts), OccupancyPyramid(L, data), pool, vol.capture_resolution,
                   vol.stats, vol.materials)


def _entry_t(camera: Camera, box, dev) -> torch.Tensor:
    """Per pixel: the primary ray's entry parameter into ``box`` (+inf if it
    misses) -- orders the ranks' segments along each ray."""
    o, d = primary_rays(camera)
    w, h = camera.resolution
    o = torch.from_numpy(np.ascontiguousarray(o)).to(dev)
    d = torch.from_numpy(np.ascontiguousarray(d)).to(dev)
    lo3 = torch.tensor(box[0], dtype=torch.float64, device=dev)
    hi3 = torch.tensor(box[1], dtype=torch.float64, device=dev)
    with np.errstate(divide="ignore"):
        inv = 1.0 / d
    t0, t1 = (lo3 - o) * inv, (hi3 - o) * inv
    tn = torch.nan_to_num(torch.minimum(t0, t1), nan=-float("inf")).amax(dim=1).clamp_min(0.0)
    tf = torch.nan_to_num(torch.maximum(t0, t1), nan=float("inf")).amin(dim=1)
    return torch.where(tn <= tf, tn, torch.full_like(tn, float("inf"))).reshape(h, w)


def render_raycast_shard(vol: FhvPofaShard, camera: Camera, lights, cfg, comm: Comm, materials=None,
                         background=(0.0, 0.0, 0.0, 0.0), *, shading: DeviceShading | None = None):
    """``render_raycast`` of the whole volume from the ranks' shards, each
    rank tracing only its own subtree (its Morton range must be one box: the
    even octant partitions, ``shard_ranges(L, N)`` for N in 1, 2, 4, 8).
    Each rank returns the full frame and its own RaycastStats.

    * opaque_nearest: each rank's first hit in its traversal order with
      alpha 1 (the kernel over a transparent background); the front-most
      region with a hit wins -- bit-identical to the 1-GPU render.
    * transparency: each rank's front-to-back partial (premultiplied C,
      coverage A), composited across ranks in entry order, then over the
      background.  Equal to the 1-GPU render up to floating-point
      reassociation when the cutoff is 1 (or off): after full coverage the
      later segments are multiplied by 1 - A = 0.  A cutoff below 1 would
      need each rank's entry coverage (not supported).
    * transparency_shadows: shadow rays cross ranks -- replicate the volume.
    """
    from .raycast import RAYCAST_MODES, default_raycast_config, render_raycast
    if cfg is None:
        cfg = default_raycast_config(vol)
    if cfg.mode == "transparency_shadows":
        raise FhvError("shadow rays cross shards: ray-cast a replicated volume for transparency_shadows")
    if cfg.mode == "transparency" and cfg.alpha_cutoff is not None and cfg.alpha_cutoff < 1.0:
        raise FhvError("sharded transparency ray cast needs alpha_cutoff 1.0 or None")
    box = region_box(vol.cell_lo, vol.cell_hi, vol.levels)
    if box is None:
        raise FhvError("this rank's Morton range is not one box: use shard_ranges(L, N) for N in 1, 2, 4, 8")
    dev = vol.pool.device
    local = local_volume(vol)
    img, st = render_raycast(local, camera, lights, cfg, materials if materials is not None else vol.materials,
                             (0.0, 0.0, 0.0, 0.0), shading=shading)
    t_in = _entry_t(camera, box, dev)
    parts = comm.all_gather_tensor(img.pixels)
    ts = torch.stack(comm.all_gather_tensor(t_in))  # [N, h, w]
    order = torch.argsort(ts, dim=0, stable=True)
    P = torch.stack(parts)  # [N, h, w, 4] premultiplied (C, A) per rank
    C = torch.zeros_like(P[0, ..., :3])
    A = torch.zeros_like(P[0, ..., 3])
    for k in range(P.shape[0]):
        pk = torch.gather(P, 0, order[k][None, ..., None].expand(1, *P.shape[1:3], 4))[0]
        C = C + (1.0 - A)[..., None] * pk[..., :3]
        A = A + (1.0 - A) * pk[..., 3]
    bg = torch.tensor(background, dtype=torch.float64, device=dev)
    out = torch.empty_like(P[0])
    if cfg.mode == "opaque_nearest":
        hit = A > 0.0
        out[..., :3] = torch.where(hit[..., None], C, bg[:3].expand_as(C))
        out[..., 3] = torch.where(hit, torch.ones_like(A), bg[3].expand_as(A))
    else:
        out[..., :3] = C + ((1.0 - A) * bg[3])[..., None] * bg[:3]
        out[..., 3] = A + (1.0 - A) * bg[3]
    img.pixels.copy_(out)
    return img, st
