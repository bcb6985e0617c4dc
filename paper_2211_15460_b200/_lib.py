"""ctypes binding of libfhv_b200.so (the C ABI declared in include/fhv_b200.h).

There is no CPU fallback: if the extension is missing or no CUDA device is
present, every entry point raises.  Build with ``python -c "import
__graft_entry__ as g; g.build()"`` (or ``python -m paper_2211_15460_b200.build``).
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FHV_LIB") or os.path.join(HERE, "libfhv_b200.so")  # FHV_LIB: experiment variants

c_i32, c_i64, c_f64, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p

FHV_OK, FHV_OVERFLOW, FHV_PASS_MISMATCH, FHV_BAD_ARGS, FHV_CUDA_ERROR = 0, 1, 2, 3, 4
FHV_RANGE, FHV_BASIS, FHV_NOMEM, FHV_TOO_MANY, FHV_SPLAT_BIG = 5, 6, 7, 8, 9
FHV_NEED_POOL = 10
FHV_STALE = 11
FHV_ALLOC_ATOMIC, FHV_EXACT_ORDER = 1, 2
FHV_SPLAT_PACKED, FHV_SPLAT_NOSYNC = 1, 2


class Tris(ctypes.Structure):
    _fields_ = [("n_tri", c_i64), ("pos", c_vp), ("vnrm", c_vp), ("fnrm", c_vp), ("mat", c_vp), ("obj", c_vp)]


class CaptureCfg(ctypes.Structure):
    _fields_ = [("strategy", c_i32), ("res", c_i32), ("pitch", c_f64), ("proj", c_f64 * 48)]


class Pool(ctypes.Structure):
    _fields_ = [("capacity", c_i64), ("pos", c_vp), ("nrm", c_vp), ("mat", c_vp), ("obj", c_vp), ("prev", c_vp)]


class Shard(ctypes.Structure):
    _fields_ = [("cell_lo", ctypes.c_uint64), ("cell_hi", ctypes.c_uint64), ("n_boxes", c_i32), ("margin", c_f64),
                ("boxes", (c_f64 * 6) * 64)]


class Shading(ctypes.Structure):
    _fields_ = [("n_lights", c_i32), ("light_kind", c_vp), ("light_vec", c_vp), ("light_color", c_vp),
                ("light_ambient", c_vp), ("n_mats", c_i32), ("diffuse", c_vp), ("specular", c_vp),
                ("shininess", c_vp), ("alpha", c_vp)]


FHV_MAX_PEERS = 8


class Peer(ctypes.Structure):
    _fields_ = [("nranks", c_i32), ("width", c_i64), ("height", c_i64), ("keys", c_vp * FHV_MAX_PEERS),
                ("winners", c_vp * FHV_MAX_PEERS), ("rgba", c_vp * FHV_MAX_PEERS), ("depth", c_vp * FHV_MAX_PEERS)]


class Volume(ctypes.Structure):
    _fields_ = [("layout", c_i32), ("levels", c_i32), ("offsets", c_vp), ("counts", c_vp), ("heads", c_vp),
                ("prev", c_vp), ("pyramid", c_vp), ("pos", c_vp), ("nrm", c_vp), ("mat", c_vp), ("obj", c_vp)]


class GBuf(ctypes.Structure):
    _fields_ = [("position", c_vp), ("normal", c_vp), ("material_id", c_vp), ("object_id", c_vp), ("valid", c_vp)]


_P = ctypes.POINTER
_SIGS = {
    "fhv_version": (ctypes.c_char_p, []),
    "fhv_ctx_create": (c_vp, []),
    "fhv_ctx_destroy": (None, [c_vp]),
    "fhv_ctx_launches": (c_i64, [c_vp]),
    "fhv_ctx_counters": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int]),
    "fhv_prof_enable": (ctypes.c_int, [c_vp, ctypes.c_int]),
    "fhv_prof_collect": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int]),
    "fhv_prof_stage_name": (ctypes.c_char_p, [ctypes.c_int]),
    "fhv_capture_list": (ctypes.c_int, [c_vp, _P(Tris), _P(CaptureCfg), c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                        _P(c_i64), c_vp]),
    "fhv_build_ppfl": (ctypes.c_int, [c_vp, _P(Tris), _P(CaptureCfg), c_i64, _P(Pool), c_vp, c_i32, _P(c_i64),
                                      c_vp]),
    "fhv_build_pofl": (ctypes.c_int, [c_vp, _P(Tris), _P(CaptureCfg), c_i32, _P(Pool), c_vp, c_vp, c_i32,
                                      _P(c_i64), c_vp]),
    "fhv_pofa_count": (ctypes.c_int, [c_vp, _P(Tris), _P(CaptureCfg), c_i32, c_vp, c_vp, c_vp, _P(c_i64), c_vp]),
    "fhv_pofa_build": (ctypes.c_int, [c_vp, _P(Tris), _P(CaptureCfg), c_i32, c_vp, c_vp, c_vp, _P(Pool), c_i32,
                                      _P(c_i64), c_vp]),
    "fhv_pofa_scatter": (ctypes.c_int, [c_vp, _P(Tris), _P(CaptureCfg), c_i32, c_vp, c_vp, _P(Pool), c_i32,
                                        c_vp]),
    "fhv_pofa_shard_count": (ctypes.c_int, [c_vp, _P(Tris), _P(CaptureCfg), c_i32, _P(Shard), c_vp, _P(c_i64),
                                            c_vp]),
    "fhv_pofa_shard_directory": (ctypes.c_int, [c_vp, c_i32, _P(Shard), c_vp, c_vp, c_vp, ctypes.c_uint64, c_vp]),
    "fhv_pofa_shard_scatter": (ctypes.c_int, [c_vp, _P(Tris), _P(CaptureCfg), c_i32, _P(Shard), c_vp, c_vp,
                                              ctypes.c_uint64, _P(Pool), c_i32, c_vp]),
    "fhv_pofa_shard_build_async": (ctypes.c_int, [c_vp, _P(Tris), _P(CaptureCfg), c_i32, _P(Shard), c_vp, c_vp, c_vp,
                                                  ctypes.c_uint64, _P(Pool), c_i32, c_vp, c_vp]),
    "fhv_splat": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_f64, c_vp, _P(Shading), c_vp, c_vp,
                                 c_vp, _P(GBuf), c_i32, c_vp]),
    "fhv_splat_shard_keys": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_f64, c_vp, c_vp, c_vp]),
    "fhv_splat_shard_winners": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_f64, c_vp, c_i64, c_vp, c_vp]),
    "fhv_splat_shard_resolve": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_f64, _P(Shading), c_vp, c_vp,
                                               c_i64, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "fhv_splat_peer": (ctypes.c_int, [c_vp, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_f64, _P(Shading), c_vp, _P(Peer),
                                      c_i32, c_i64, c_vp, c_vp]),
    "fhv_raycast": (ctypes.c_int, [c_vp, _P(Volume), _P(Shading), c_vp, c_vp, c_f64, c_f64, c_i32, c_f64, c_i64,
                                   c_i64, c_vp, c_vp, c_vp, c_vp]),
    "fhv_raycast_image": (ctypes.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, _P(Volume), _P(Shading), c_vp, c_vp,
                                         c_f64, c_f64, c_i32, c_f64, c_vp, c_vp, c_vp, c_vp]),
    "fhv_rebuild_pofa": (ctypes.c_int, [c_vp, c_i32, _P(Pool), c_i64, c_vp, c_vp, c_vp, _P(Pool), c_vp]),
    "fhv_pack_records": (ctypes.c_int, [c_vp, _P(Pool), c_i64, c_vp, c_vp]),
    "fhv_unpack_records": (ctypes.c_int, [c_vp, c_vp, c_i64, _P(Pool), c_vp]),
    "fhv_selftest_div": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "fhv_unit_rows": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, _P(c_i64), c_vp]),
    "fhv_deferred": (ctypes.c_int, [c_vp, _P(Tris), c_vp, c_i32, c_i32, c_vp, _P(Shading), c_vp, c_vp, c_vp,
                                    _P(GBuf), _P(c_i64), c_vp]),
    "fhv_face_normals": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp]),
    "fhv_expand_indexed": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "fhv_capture_list_depth": (ctypes.c_int, [c_vp, _P(Tris), _P(CaptureCfg), c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                              c_vp, _P(c_i64), c_vp]),
    "fhv_raster_screen": (ctypes.c_int, [c_vp, _P(Tris), c_vp, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                         c_vp, _P(c_i64), c_vp]),
    "fhv_op_coverage": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       _P(c_i64), _P(c_i64), c_vp]),
    "fhv_op_linked_insert": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp]),
    "fhv_op_pofa_scatter": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, _P(c_i64), c_vp]),
    "fhv_pofa_build_async": (ctypes.c_int, [c_vp, _P(Tris), _P(CaptureCfg), c_i32, c_vp, c_vp, c_vp, _P(Pool), c_i32,
                                            c_vp, c_vp]),
    "fhv_build_pofl_async": (ctypes.c_int, [c_vp, _P(Tris), _P(CaptureCfg), c_i32, _P(Pool), c_vp, c_vp, c_i32, c_vp,
                                            c_vp]),
    "fhv_ticket_check": (ctypes.c_int, [c_vp, c_i64]),
    "fhv_ticket_accumulate": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp]),
    "fhv_chain_indices": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp, _P(c_i64), c_vp]),
    "fhv_set_paths": (ctypes.c_int, [c_vp, c_i32, c_i64, c_vp, c_vp, c_vp]),
    "fhv_pyramid_from_occupancy": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp]),
    "fhv_project_points": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "fhv_shade": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, _P(Shading), c_vp, c_vp, c_vp]),
    "fhv_ray_probe": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, _P(Volume), _P(Shading), c_vp, c_vp,
                                     c_f64, c_f64, c_i32, c_f64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "fhv_transmittance": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i32, c_vp, c_vp, _P(Volume), _P(Shading), c_f64,
                                         c_f64, c_vp, c_vp, c_vp]),
    "fhv_leaf_order": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_f64, c_f64, c_i64, c_vp, c_vp, c_vp, c_vp,
                                      c_vp]),
    "fhv_intersect_points": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_f64, c_f64, c_f64, c_vp, c_vp, c_vp]),
}
EXPORTED = tuple(_SIGS)

_lib = None
_ctxs: dict = {}
_lock = threading.Lock()


class ExtensionMissing(RuntimeError):
    pass


def load(require_cuda: bool = True):
    """Load the shared library (idempotent).  Raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissing(f"{LIB_PATH} not built; run __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_cuda and not torch.cuda.is_available():
        raise RuntimeError("fhv_b200 needs a CUDA device (B200); there is no CPU fallback")
    return _lib


def ctx(device: torch.device):
    """Scratch context of (device, calling host thread, current stream),
    created on first use.  A context is single-stream (the header's contract:
    its control block and scratch are reused call after call), so host
    threads that share a device -- e.g. the loopback shards of
    shard.ThreadComm -- and work issued on different streams of one thread --
    e.g. a capture overlapping the previous step's splat -- each get their own."""
    lib = load()
    idx = device.index if device.index is not None else torch.cuda.current_device()
    key = (idx, threading.get_ident(), torch.cuda.current_stream(idx).cuda_stream)
    with _lock:
        c = _ctxs.get(key)
        if c is None:
            with torch.cuda.device(idx):
                c = lib.fhv_ctx_create()
            if not c:
                raise MemoryError("fhv_ctx_create failed")
            if _prof_on.get(idx):
                lib.fhv_prof_enable(c, 1)
            _ctxs[key] = c
            if threading.current_thread() is not threading.main_thread() and not hasattr(_tls, "reaper"):
                _tls.reaper = _ThreadReaper(threading.get_ident())
    return c


_tls = threading.local()
_retired: dict = {}  # device index -> launches of destroyed contexts (launch accounting survives release)


def release(device: torch.device | None = None, thread_id: int | None = None, stream=None) -> int:
    """Destroy the scratch contexts matching (device, host thread, stream)
    (None = any) and free their grow-only scratch; returns how many.  Contexts
    of a worker thread are released automatically when the thread ends."""
    idx = None
    if device is not None:
        idx = device.index if device.index is not None else torch.cuda.current_device()
    sptr = stream.cuda_stream if stream is not None and hasattr(stream, "cuda_stream") else stream
    lib = load(require_cuda=False)
    with _lock:
        keys = [k for k in _ctxs if (idx is None or k[0] == idx) and (thread_id is None or k[1] == thread_id)
                and (sptr is None or k[2] == sptr)]
        gone = [(k, _ctxs.pop(k)) for k in keys]
    for k, c in gone:
        _retired[k[0]] = _retired.get(k[0], 0) + int(lib.fhv_ctx_launches(c))
        lib.fhv_ctx_destroy(c)
    return len(gone)


class _ThreadReaper:
    """Thread-local sentinel: collected when its thread exits, releasing the
    contexts that thread created."""

    def __init__(self, tid: int):
        self.tid = tid

    def __del__(self):
        try:
            release(thread_id=self.tid)
        except Exception:  # interpreter shutdown
            pass


_prof_on: dict = {}


def _device_ctxs(device: torch.device) -> list:
    ctx(device)  # at least the current one
    idx = device.index if device.index is not None else torch.cuda.current_device()
    with _lock:
        return [c for k, c in _ctxs.items() if k[0] == idx]


def launches(device: torch.device) -> int:
    """Kernel launches issued through this library on the device (all contexts)."""
    lib = load()
    idx = device.index if device.index is not None else torch.cuda.current_device()
    return int(sum(lib.fhv_ctx_launches(c) for c in _device_ctxs(device))) + _retired.get(idx, 0)


def counters(device: torch.device) -> tuple:
    """(re-sorted by the tile pass, reserved, long leaves listed for the
    per-leaf pass) of the last synchronised EXACT_ORDER POFA build on the
    calling thread's current context (fhv_ctx_counters)."""
    import numpy as np
    out = np.zeros(3, dtype=np.int64)
    load().fhv_ctx_counters(ctx(device), out.ctypes.data, 3)
    return tuple(int(v) for v in out)


def raycast_diag(device: torch.device) -> tuple:
    """(rays handed to the per-ray kernel, (ray, node) pairs that took their
    own child order) of the last packet ray cast on the calling thread's
    context (fhv_ctx_counters words 3-4; synchronises the device)."""
    import numpy as np
    out = np.zeros(5, dtype=np.int64)
    rc = load().fhv_ctx_counters(ctx(device), out.ctypes.data, 5)
    if rc < 0:
        check(-rc, "raycast_diag")
    return int(out[3]), int(out[4])


def prof_enable(device: torch.device, on: bool = True) -> None:
    idx = device.index if device.index is not None else torch.cuda.current_device()
    _prof_on[idx] = on
    for c in _device_ctxs(device):
        load().fhv_prof_enable(c, 1 if on else 0)


def prof_collect(device: torch.device) -> dict:
    """{stage: (total_ms, launches)} since the last collect, over every
    context of the device (syncs)."""
    import numpy as np
    lib = load()
    out: dict = {}
    for c in _device_ctxs(device):
        ms = np.zeros(64)
        cnt = np.zeros(64, dtype=np.int64)
        n = lib.fhv_prof_collect(c, ms.ctypes.data, cnt.ctypes.data, 64)
        for i in range(n):
            if cnt[i]:
                name = lib.fhv_prof_stage_name(i).decode()
                t, k = out.get(name, (0.0, 0))
                out[name] = (t + float(ms[i]), k + int(cnt[i]))
    return out


def stream_ptr(device: torch.device):
    return c_vp(torch.cuda.current_stream(device).cuda_stream)


_ctx_fast: dict = {}


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return c_vp(t.data_ptr()) if t.numel() else None


def check(rc: int, what: str, allow=(FHV_OK,)):
    """Map an FHV_* status to the reference's exception types."""
    if rc in allow:
        return rc
    from .scene import SceneError
    from .storage import FhvError, PofaBuildError
    msg = f"{what}: status {rc}"
    if rc == FHV_PASS_MISMATCH:
        raise PofaBuildError(f"{what}: per-octant cursors do not match counted sizes")
    if rc == FHV_RANGE:
        raise FhvError(f"{what}: position outside [0,1]^3")
    if rc == FHV_BASIS:
        raise ValueError(f"{what}: tangent_basis received a non-unit normal")
    if rc == FHV_TOO_MANY:
        raise FhvError(f"{what}: fragment count exceeds 32-bit directory range")
    if rc == FHV_SPLAT_BIG:
        raise SceneError("splat footprint too large; reduce the radius")
    if rc == FHV_NOMEM:
        raise MemoryError(msg)
    if rc == FHV_BAD_ARGS:
        raise FhvError(f"{what}: invalid arguments")
    raise RuntimeError(msg)
