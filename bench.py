#!/usr/bin/env python
"""Benchmark of the FHV hot path on B200: capture + novel-view reconstruction.

Workload (default --config C3): ``scatter1M`` -- 48
icospheres, 983,040 triangles, synthetic (seeded; byte-identical to the same
field built by the reference's own ``icosphere`` / ``make_triangle``,
tests/test_scene_pinning.py), captured with the NormalSpace strategy at
pitch 1/1080 into a POFA octree of depth 8 (two-pass count / scan / scatter,
the reference's exact in-leaf order by default), then one 1920x1080
perspective novel view reconstructed by exact z-tested point splatting.  One
step = capture + one reconstruct.  ``value`` = fragments captured per second
of step time (inputs resident in HBM); ``e2e`` = the same through the public
API with the scene copied host->device (pinned) and the image copied back
every step; ``parity`` = the last timed step's pool and image against the
oracle port on the same inputs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--fast-order]

--impl reference times the reference algorithm's CPU implementation (the
oracle port, oracle/fhv_oracle.c, bit-identical to the reference's golden
vectors) on ALL the host's threads (the port parallelises the capture and
splat without changing their results; the shipped reference, fastest at
threads=1, runs ~6.5 k frag/s -- ~575x below the port on one thread, ~1,650x
below it on 16: profiles/r02_shipped_reference.json) on the same workload
and prints the same JSON line shape and ``config``.
Multi-GPU (torchrun, N>1): the same scene is partitioned by Morton range
(paper_2211_15460_b200/shard.py): each rank bins the
triangles of its leaf range, captures its slice of the POFA (after the first
step with no host wait and no collective: every rank's total, hence its
global base, speculated from the previous build, all ranks' tickets checked
after the timed loop) and splats its fragments; the frame is composited by
depth (NVLink peer-memory slabs, or NCCL all-reduces).  Strong scaling: fixed total work; time = max over ranks;
value = all fragments / that time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0
METRIC = "fragments captured/s + novel-view frames/s at 1080p (GB/s vs HBM peak)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--config", default="C3", choices=("C3", "C2", "C4", "C5"),
                    help="C3 = the headline workload; C2 / C4 / C5 = the other BASELINE configs (1 GPU)")
    ap.add_argument("--fast-order", dest="exact_order", action="store_false",
                    help="the paper's atomic in-leaf POFA order (per-leaf multiset equal) instead of the reference's "
                         "exact order (default: exact, byte-identical pool)")
    ap.add_argument("--exact-order", dest="exact_order", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--packed", action="store_true", help="packed 64-bit splat z-test")
    ap.add_argument("--c5-partition", default="views", choices=("views", "subtrees"),
                    help="C5 on N GPUs: shard the 64 views (POFA replicated) or the octree (each rank traces its "
                         "octant subtrees of every view; partials composited in entry order)")
    ap.add_argument("--composite", default="auto", choices=("auto", "peer", "allreduce"),
                    help="multi-GPU splat composite: peer memory (fhv_splat_peer over NVLink P2P) or NCCL "
                         "all-reduces; auto = peer when the peer mappings can be set up")
    ap.add_argument("--no-graph", action="store_true",
                    help="time the Python-enqueued steps instead of CUDA-graph replays of one captured step")
    ap.add_argument("--sync-steps", action="store_true",
                    help="wait for each pofa_build on the host (default: asynchronous steps, tickets checked)")
    ap.add_argument("--upload", default="indexed", choices=("indexed", "soup"),
                    help="e2e: the scene crosses PCIe as an indexed mesh expanded on the device (default) or as the "
                         "triangle arrays")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="few steps, no clocks/e2e/cpu (for ncu)")
    return ap.parse_args()


def peaks():
    try:
        m = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


# ---------------------------------------------------------------------------
# workload


def workload():
    from paper_2211_15460_b200 import sample_scenes
    from paper_2211_15460_b200.lights import headlight
    from paper_2211_15460_b200.raster import CaptureStrategy, RasterConfig
    from paper_2211_15460_b200.scene import capture_camera, viewpoint_camera
    scene = sample_scenes.scatter1m()
    cam = capture_camera(scene, "+z", 1080)
    cfg = RasterConfig((1920, 1080), RasterConfig.from_camera(cam).projection, extent=1.0)
    view = viewpoint_camera("+x", (1920, 1080), "perspective")
    return {"scene": scene, "cfg": cfg, "strategy": CaptureStrategy.normal_space(), "levels": 8, "view": view,
            "lights": [headlight(view)], "radius": 1.0 / 1080}


CONFIG = {"workload": "C3 scatter1M: 983,040 tris, NormalSpace capture pitch 1/1080 -> POFA L=8, "
                      "+ 1920x1080 perspective splat reconstruct",
          "triangles": 983040, "capture_res": 1080, "levels": 8, "view": [1920, 1080],
          "l2_note": "inputs + outputs per step (~0.9 GB) exceed the 126 MB L2"}


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML)


class ClockSampler:
    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.02)  # sparse: NVML queries take driver locks the launching thread also needs

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


# ---------------------------------------------------------------------------
# CPU baseline / reference arm (oracle port)


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_run(w, threads: int = 1, keep: bool = False):
    """One full C3 step on the host with the oracle port: POFA capture + the
    1080p splat, on ``threads`` host threads (threads=1 is the reference's
    sequential order; more threads keep the directory and image identical).
    ``keep``: also return (volume, rgba, depth) for the parity check."""
    from oracle import oracle as orc
    with orc.threads(threads):
        t0 = time.perf_counter()
        vol = orc.pofa_build(w["scene"], w["strategy"], w["cfg"], w["levels"])
        t1 = time.perf_counter()
        rgba, depth, _ = orc.splat(vol["pool"], vol["next_free"], w["view"], w["lights"], w["radius"],
                                   w["scene"].materials)
        t2 = time.perf_counter()
    if keep:
        return vol["next_free"], t1 - t0, t2 - t1, (vol, rgba, depth)
    return vol["next_free"], t1 - t0, t2 - t1


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = workload()
    nt = host_threads()
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_run(w, nt)
    tot_s, frags = 0.0, 0
    steps = min(args.steps, 30)  # each step ~0.5-2 s of host time; keep the arm within a few minutes
    for _ in range(steps):
        n, tc, ts = cpu_run(w, nt)
        tot_s += tc + ts
        frags += n
    value = frags / tot_s
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "frag/s", "n_gpus": args.gpus,
            "steps": steps, "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded icosphere field)", "config": CONFIG,
            "cpu_baseline": {"value": value, "unit": "frag/s", "cores": nt, "kind": "port",
                             "sample": f"{steps} full C3 steps (POFA capture + 1080p splat), oracle/fhv_oracle.c "
                                       f"on {nt} host threads"},
            "e2e": {"value": value, "unit": "frag/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm


# ---------------------------------------------------------------------------
# the other BASELINE configs, one GPU


def _timed(fn, steps, stream):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    out = None
    for _ in range(steps):
        out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, out


def _stage_profile(fn, steps, dev):
    from paper_2211_15460_b200 import _lib
    _lib.prof_enable(dev, True)
    _lib.prof_collect(dev)
    for _ in range(steps):
        fn()
    import torch
    torch.cuda.synchronize()
    prof = _lib.prof_collect(dev)
    _lib.prof_enable(dev, False)
    return {k: v[0] / steps for k, v in prof.items()}, prof


def extra_config(args):
    """C2: spheres100k POFL L8 capture + 1080p ray-cast view; C4: layers80
    depth-complex 1080^2 PPFL vs POFA; C5: 64 4K ray-cast views of C3's POFA."""
    import numpy as np
    import torch
    import paper_2211_15460_b200 as fhv
    from paper_2211_15460_b200 import _lib, sample_scenes
    from paper_2211_15460_b200.device import DeviceShading, device_scene
    from paper_2211_15460_b200.lights import ImageBuffer, headlight
    from paper_2211_15460_b200.raster import CaptureStrategy, RasterConfig
    from paper_2211_15460_b200.scene import capture_camera, viewpoint_camera
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("FHV_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    if world > 1 and args.config != "C5":
        raise SystemExit("--config C2 / C4 run on one GPU (C4's PPFL is view-bound: replicas only)")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import torch.distributed as dist
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    stream = torch.cuda.current_stream(dev)
    peak, peak_kind = peaks()
    ns = CaptureStrategy.normal_space()
    nt = host_threads()
    line = {"metric": METRIC, "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, no dataset)", "scaling": "strong", "higher_is_better": True}

    def ray_bytes(st, P):  # 16 tested + 8 visited + 20 hits + 32 P
        return 16 * st.tested_fragments + 8 * st.visited_leaves + 20 * st.hits + 32 * P

    def img_buf(w, h):
        return ImageBuffer(w, h, torch.empty((h, w, 4), dtype=torch.float64, device=dev),
                           torch.empty((h, w), dtype=torch.float64, device=dev))

    if args.config == "C2":
        scene = sample_scenes.spheres100k()
        cam = capture_camera(scene, "+z", 1080)
        cfg = RasterConfig((1920, 1080), RasterConfig.from_camera(cam).projection, extent=1.0)
        view = viewpoint_camera("+x", (1920, 1080), "perspective")
        lights = [headlight(view)]
        ds = device_scene(scene, dev)
        sh = DeviceShading(scene.materials, lights, dev)
        buf = img_buf(1920, 1080)
        vol0 = fhv.build_pofl(scene, ns, cfg, 8, device=dev)
        rcfg = fhv.default_raycast_config(vol0)

        n0 = vol0.pool.next_free
        acc2 = torch.zeros(2, dtype=torch.int64, device=dev)
        tk2 = torch.zeros(4, dtype=torch.int64).pin_memory()

        def step():
            # asynchronous POFL build (no host wait; its ticket checked on the
            # device) and the ray cast of the same stream
            vol = fhv.build_pofl(scene, ns, cfg, 8, device=dev, sync=False, ticket=tk2)
            _lib.check(_lib.load().fhv_ticket_accumulate(_lib.ctx(dev), int(n0), _lib.ptr(acc2),
                                                         _lib.stream_ptr(dev)), "ticket")
            # (every pixel is written by the cast: the buffer is reused as is)
            img, st = fhv.render_raycast(vol, view, lights, rcfg, out=buf, sync=False, shading=sh)
            return vol, st
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        g2 = None
        if not args.no_graph:  # the step captured once in a CUDA graph and replayed
            gs2 = torch.cuda.Stream(dev)
            with torch.cuda.stream(gs2):
                for _ in range(2):
                    step()
            torch.cuda.synchronize()
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2, stream=gs2):
                g_out = step()
            torch.cuda.synchronize()
            g2.replay()
            torch.cuda.synchronize()
        acc2.zero_()
        with ClockSampler(0) as clk:
            if g2 is not None:
                ms, _ = _timed(g2.replay, args.steps, stream)
                vol, st = g_out
            else:
                ms, (vol, st) = _timed(step, args.steps, stream)
        bad2, checked2 = (int(v) for v in acc2.cpu().tolist())
        if bad2 or checked2 != args.steps:
            raise RuntimeError(f"C2 steps: build ticket status {bad2}, {checked2}/{args.steps} checked")
        stats = fhv.RaycastStats(*st.counters.cpu().tolist())
        n = n0
        stage, prof = _stage_profile(step, args.steps, dev)
        t_ray = stage.get("raycast", 0.0) + stage.get("raycast_handoff", 0.0)  # packet + per-ray hand-off kernels
        P = 1920 * 1080
        rb = ray_bytes(stats, P)
        line.update({"value": n / (ms / 1e3), "unit": "frag/s", "ms_per_step": ms,
                     "config": {"workload": "C2 spheres100k: 102,400 tris, NormalSpace pitch 1/1080 -> POFL L=8 "
                                            "(linked lists), + 1920x1080 perspective ray-cast (transparency, "
                                            "cutoff 1.0)", "fragments": n, "parallelism": "single"},
                     "novel_view_fps": 1e3 / t_ray if t_ray else None, "raycast_stats": stats.as_dict(),
                     "stage_ms": {k: round(v, 4) for k, v in sorted(stage.items(), key=lambda kv: -kv[1])},
                     "roofline": {"bound": "hbm", "kernel": "raycast", "achieved": round(rb / (t_ray / 1e3) / 1e9, 1),
                                  "peak": peak, "unit": "GB/s", "frac": round(rb / (t_ray / 1e3) / 1e9 / peak, 4),
                                  "traffic": None, "algorithmic_bytes": rb, "peak_kind": peak_kind,
                                  "note": "packet traversal, latency bound (register-limited occupancy), see "
                                          "profiles/"},
                     "host": ("CUDA-graph replays of one captured step (asynchronous POFL build + ray cast), every "
                              "build ticket checked on the device" if g2 is not None else
                              "Python-enqueued asynchronous steps, build tickets checked on the device"),
                     "clocks": clk.summary()})
        if not args.no_cpu_baseline:
            from oracle import oracle as orc
            with orc.threads(nt):
                t0 = time.perf_counter()
                rv = orc.build_pofl(scene, ns, cfg, 8)
                t1 = time.perf_counter()
            band = (480, 600)  # 120 of 1080 rows, scaled x9
            orc.raycast(rv, view, lights, rcfg.splat_radius_world, materials=scene.materials, rows=band)
            t2 = time.perf_counter()
            tr = (t2 - t1) * 1080 / (band[1] - band[0])
            line["cpu_baseline"] = {"value": rv["next_free"] / (t1 - t0 + tr), "unit": "frag/s", "cores": nt,
                                    "kind": "port", "sample": f"POFL capture ({nt} threads) {t1 - t0:.2f} s + "
                                    f"ray-cast rows {band} (1 thread) scaled to 1080 rows = {tr:.2f} s",
                                    "novel_view_fps": 1.0 / tr}
    elif args.config == "C4":
        scene = sample_scenes.layers80()
        cfg = RasterConfig.from_camera(capture_camera(scene, "+z", 1080))
        one = CaptureStrategy.one_view()
        device_scene(scene, dev)
        n = fhv.pofa_build(scene, one, cfg, 8, device=dev).pool.next_free

        def step_pofa():
            return fhv.pofa_build(scene, one, cfg, 8, device=dev)

        def step_ppfl():
            return fhv.build_ppfl(scene, cfg, one, capacity=n, device=dev)
        for _ in range(args.warmup):
            step_pofa()
            step_ppfl()
        # the POFA step as C3 times it: the asynchronous build (pool sized by
        # the last exact total, no host wait) captured once in a CUDA graph
        # and replayed; every replay's build ticket is checked on the device
        ds4 = device_scene(scene, dev)
        acc4 = torch.zeros(2, dtype=torch.int64, device=dev)
        tk4 = torch.zeros(4, dtype=torch.int64).pin_memory()
        gs4 = torch.cuda.Stream(dev)

        def step_pofa_async():
            v = fhv.pofa_build(scene, one, cfg, 8, device=dev, tris=ds4, sync=False, ticket=tk4)
            _lib.check(_lib.load().fhv_ticket_accumulate(_lib.ctx(dev), int(n), _lib.ptr(acc4),
                                                         _lib.stream_ptr(dev)), "ticket")
            return v
        g4 = None
        if not args.no_graph:
            with torch.cuda.stream(gs4):
                for _ in range(2):
                    step_pofa_async()
            torch.cuda.synchronize()
            g4 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g4, stream=gs4):
                step_pofa_async()
            torch.cuda.synchronize()
            g4.replay()
            torch.cuda.synchronize()
            acc4.zero_()
        with ClockSampler(0) as clk:
            if g4 is not None:
                ms_a, _ = _timed(g4.replay, args.steps, stream)
                bad4, checked4 = (int(v) for v in acc4.cpu().tolist())
                if bad4 or checked4 != args.steps:
                    raise RuntimeError(f"C4 graph replays: build ticket status {bad4}, {checked4}/{args.steps}")
            else:
                ms_a, _ = _timed(step_pofa, args.steps, stream)
            ms_sync, _ = _timed(step_pofa, args.steps, stream)
            ms_p, _ = _timed(step_ppfl, args.steps, stream)
        st_a, _ = _stage_profile(step_pofa, args.steps, dev)
        st_p, _ = _stage_profile(step_ppfl, args.steps, dev)
        mem_a = fhv.memory_report("POFA", levels=8, exact_count=n, record_size=36)["total_bytes"]
        mem_p = fhv.memory_report("PPFL", resolution=(1080, 1080), capacity=n, record_size=36)["total_bytes"]
        dom = max(st_a, key=st_a.get)
        T = scene.n_triangles
        algo = {"emit_pofa": 176 * T + 36 * n, "count_leaves": 72 * T + 4 * 8 ** 8,
                "scan_leaves": 8 * 8 ** 8 + 8 ** 7}.get(dom)
        line.update({"value": n / (ms_a / 1e3), "unit": "frag/s", "ms_per_step": ms_a,
                     "config": {"workload": "C4 layers80: 80 translucent quads, 1080^2 OneView capture, POFA L=8 "
                                            "(value) vs PPFL with explicit capacity", "fragments": n,
                                "parallelism": "single"},
                     "ppfl": {"value": n / (ms_p / 1e3), "unit": "frag/s", "ms_per_step": ms_p, "bytes": mem_p,
                              "stage_ms": {k: round(v, 4) for k, v in st_p.items()}},
                     "pofa": {"bytes": mem_a, "stage_ms": {k: round(v, 4) for k, v in st_a.items()},
                              "host": ("CUDA-graph replays of one captured asynchronous build, every build ticket "
                                       "checked on the device" if g4 is not None else "Python-enqueued sync builds"),
                              "sync_build_ms_per_step": ms_sync},
                     "clocks": clk.summary()})
        if algo:
            t = st_a[dom] / 1e3
            line["roofline"] = {"bound": "hbm", "kernel": dom, "achieved": round(algo / t / 1e9, 1), "peak": peak,
                                "unit": "GB/s", "frac": round(algo / t / 1e9 / peak, 4), "traffic": None,
                                "algorithmic_bytes": algo, "peak_kind": peak_kind}
        if not args.profile_only:
            # SURVEY.md section 8(d) C4 "optional raycast R/T": one 1080p
            # perspective view through all 80 translucent layers of the POFA
            vol4 = fhv.pofa_build(scene, one, cfg, 8, device=dev)
            view4 = viewpoint_camera("+z", (1920, 1080), "perspective")
            rc4 = fhv.default_raycast_config(vol4)
            sh4 = DeviceShading(scene.materials, [headlight(view4)], dev)
            buf4 = img_buf(1920, 1080)

            def step_ray4():
                return fhv.render_raycast(vol4, view4, [headlight(view4)], rc4, out=buf4, sync=False, shading=sh4)[1]
            step_ray4()
            ms_r, st4 = _timed(step_ray4, max(1, min(args.steps, 5)), stream)
            line["raycast"] = {"value": 1e3 / ms_r, "unit": "frames/s", "ms_per_view": ms_r,
                               "view": "viewpoint_camera('+z', 1920x1080, perspective), transparency, cutoff 1.0",
                               "raycast_stats": fhv.RaycastStats(*st4.counters.cpu().tolist()).as_dict()}
    else:  # C5
        scene = sample_scenes.scatter1m()
        cam = capture_camera(scene, "+z", 1080)
        cfg = RasterConfig((1920, 1080), RasterConfig.from_camera(cam).projection, extent=1.0)
        all_views = sample_scenes.c5_views(64)
        subtrees = args.c5_partition == "subtrees" and world > 1
        if subtrees:
            # each rank owns whole octant subtrees (one box
            # per rank), traces them for every view; per-ray (C, A) partials are
            # composited across ranks in entry order (shard.render_raycast_shard)
            from paper_2211_15460_b200 import shard as shard_mod
            comm = shard_mod.TorchComm(device=dev)
            vol = shard_mod.pofa_build_shard(scene, ns, cfg, 8, comm, balance=False, device=dev)
            rcfg = fhv.default_raycast_config(vol)
            views = all_views
            W, H = views[0].resolution
            shs = [DeviceShading(scene.materials, [headlight(v)], dev) for v in views]

            def step():
                sts = []
                for v, sh in zip(views, shs):
                    _, st = shard_mod.render_raycast_shard(vol, v, [headlight(v)], rcfg, comm, shading=sh)
                    sts.append(torch.tensor(list(st.as_dict().values()), dtype=torch.int64, device=dev))
                return sts
        else:
            # views shard across ranks, the FHV replicated
            vol = fhv.pofa_build(scene, ns, cfg, 8, device=dev)
            rcfg = fhv.default_raycast_config(vol)
            views = all_views[rank::world]
            W, H = views[0].resolution
            shs = [DeviceShading(scene.materials, [headlight(v)], dev) for v in views]
            buf = img_buf(W, H)

            def step():
                sts = []
                for v, sh in zip(views, shs):
                    _, st = fhv.render_raycast(vol, v, [headlight(v)], rcfg, out=buf, sync=False, shading=sh)
                    sts.append(st.counters)
                return sts
        for _ in range(args.warmup):
            step()
        if world > 1:
            dist.barrier()
        with ClockSampler(local) as clk:
            ms, sts = _timed(step, args.steps, stream)
        if world > 1:  # max over ranks, on the device clock
            t = torch.tensor([ms], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        tot = torch.stack(sts).sum(0).cpu().tolist()
        stats = fhv.RaycastStats(*tot)
        stage, _ = _stage_profile(step, 1, dev)
        P = W * H * len(views)
        rb = ray_bytes(stats, P)  # per step (this rank's views)
        t_ray = stage.get("raycast", ms) + stage.get("raycast_handoff", 0.0)
        line.update({"value": len(all_views) / (ms / 1e3), "unit": "frames/s", "ms_per_step": ms,
                     "rays_per_s": W * H * len(all_views) / (ms / 1e3),
                     "config": {"workload": "C5: 64 x 3840x2160 perspective ray-cast views (Fibonacci sphere, "
                                            "distance 1.5, fov 45) of C3's POFA (scatter1M, L=8)",
                                "fragments": vol.total if subtrees else vol.pool.next_free, "views": len(all_views),
                                "parallelism": (f"octant subtrees x{world}, partials composited in entry order"
                                                if subtrees else f"views sharded x{world}, FHV replicated")
                                if world > 1 else "single"},
                     "raycast_stats": stats.as_dict(),
                     "stage_ms": {k: round(v, 4) for k, v in stage.items()},
                     "roofline": {"bound": "hbm", "kernel": "raycast", "achieved": round(rb / (t_ray / 1e3) / 1e9, 1),
                                  "peak": peak, "unit": "GB/s", "frac": round(rb / (t_ray / 1e3) / 1e9 / peak, 4),
                                  "traffic": None, "algorithmic_bytes": rb, "peak_kind": peak_kind,
                                  "note": "packet traversal, latency bound (register-limited occupancy), see "
                                          "profiles/"},
                     "clocks": clk.summary()})
        if not subtrees and not args.profile_only:
            # SURVEY.md section 8(d) C5 "(and splat)": the same views reconstructed
            # by exact z-tested splatting (r = 1/1080, C3's capture pitch)
            sbuf = img_buf(W, H)

            def step_splat():
                for v, sh in zip(views, shs):
                    fhv.splat_render(vol.pool, v, [headlight(v)], 1.0 / 1080, scene.materials, out=sbuf, shading=sh)
            for _ in range(max(1, args.warmup)):
                step_splat()
            ms_s, _ = _timed(step_splat, args.steps, stream)
            if world > 1:
                t = torch.tensor([ms_s], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms_s = float(t.item())
            sst, _ = _stage_profile(step_splat, 1, dev)
            line["splat"] = {"value": len(all_views) / (ms_s / 1e3), "unit": "frames/s", "ms_per_step": ms_s,
                             "stage_ms": {k: round(v, 4) for k, v in sst.items()},
                             "note": "64 x 3840x2160 exact splats of the same POFA (depth pass, index pass, "
                                     "resolve per view)"}
        if not args.no_cpu_baseline and rank == 0 and world == 1:
            from oracle import oracle as orc
            ref = orc.pofa_build(scene, ns, cfg, 8)
            band = (1040, 1120)  # 80 of 2160 rows of view 0, scaled x27 x64
            t0 = time.perf_counter()
            orc.raycast(ref, views[0], [headlight(views[0])], rcfg.splat_radius_world, materials=scene.materials,
                        rows=band)
            dt = (time.perf_counter() - t0) * H / (band[1] - band[0])
            line["cpu_baseline"] = {"value": 1.0 / dt, "unit": "frames/s", "cores": 1, "kind": "port",
                                    "sample": f"rows {band} of one 4K view (1 thread), scaled to a full view: "
                                              f"{dt:.2f} s per view"}
    line["gpu_launches_total"] = _lib.launches(dev)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    if args.config != "C3":
        return extra_config(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2211_15460_b200 as fhv
    from paper_2211_15460_b200 import _lib
    from paper_2211_15460_b200.device import DeviceScene, DeviceShading, device_scene
    from paper_2211_15460_b200.lights import ImageBuffer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FHV_BENCH_BACKEND=gloo: functional check of the multi-rank path on fewer
    # GPUs than ranks (ranks share devices; host-staged collectives) -- never a
    # performance number
    backend = os.environ.get("FHV_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def all_max(t):
        if backend == "nccl":
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return t
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX)
        return h

    w = workload()
    scene, cfg, strat, L, view = w["scene"], w["cfg"], w["strategy"], w["levels"], w["view"]
    ds = device_scene(scene, dev)
    shading = DeviceShading(scene.materials, w["lights"], dev)
    W, H = view.resolution
    img = ImageBuffer(W, H, torch.empty((H, W, 4), dtype=torch.float64, device=dev),
                      torch.empty((H, W), dtype=torch.float64, device=dev))

    if world > 1:
        from paper_2211_15460_b200 import shard
        comm = shard.TorchComm(device=dev)
        ranges = shard.shard_ranges(L, world, shard.fragment_weights(scene, strat, cfg, L))
        bufs = shard.SplatBuffers(W, H, dev)
        peer, composite = None, args.composite
        if composite != "allreduce":
            try:  # NVLink peer mappings of every rank's splat buffers (symmetric memory)
                peer = shard.PeerFrame(W, H, comm, dev)
                composite = "peer"
            except Exception as e:  # noqa: BLE001
                if composite == "peer":
                    raise
                composite = f"allreduce (peer mapping unavailable: {type(e).__name__})"
        mode = "peer" if peer is not None else "allreduce"
        # after the first (synchronous) build every step's build is
        # speculative: no host wait and no collective (every rank's total,
        # base and binning from that build); the tickets of all ranks are
        # checked after the timed loop -- a wrong speculation fails the run
        sh_tickets = torch.zeros((4 * (args.steps + 4), 4), dtype=torch.int64).pin_memory()
        sh_used: list = []

        def step(tris=ds, out=img):
            asynchronous = not args.sync_steps and len(sh_used) < len(sh_tickets)
            tk = sh_tickets[len(sh_used)] if asynchronous else None
            vol = shard.pofa_build_shard(scene, strat, cfg, L, comm, ranges=ranges, exact_order=args.exact_order,
                                         device=dev, tris=tris, sync=not asynchronous, ticket=tk)
            if vol.pending is not None:
                sh_used.append(vol.pending[:2])
            shard.splat_render_shard(vol, view, w["lights"], w["radius"], scene.materials, comm, out=out,
                                     shading=shading, buffers=bufs, composite=mode, peer=peer)
            return vol
    else:
        composite = None
        # single GPU: after the warm-up every step is enqueued without a host
        # wait (pofa_build(sync=False): pool sized by the previous exact total,
        # outcome in a pinned ticket); every ticket of a timed loop is checked
        # after its closing sync -- a wrong speculation fails the run
        tickets = torch.zeros((4 * (args.steps + 4), 4), dtype=torch.int64).pin_memory()
        used: list = []

        def step(tris=ds, out=img):
            asynchronous = not args.sync_steps and len(used) < len(tickets)
            tk = tickets[len(used)] if asynchronous else None
            vol = fhv.pofa_build(scene, strat, cfg, L, exact_order=args.exact_order, device=dev, tris=tris,
                                 sync=not asynchronous, ticket=tk)
            if vol.pending is not None:
                used.append(vol.pending[:2])  # the ticket only: volumes are freed step by step
            fhv.splat_render(vol.pool, view, w["lights"], w["radius"], scene.materials, out=out, packed=args.packed,
                             shading=shading)
            return vol

        def check_tickets():
            torch.cuda.synchronize()
            for tk, guess in used:
                rc = fhv.storage.ticket_status(tk, guess)
                if rc != 0:
                    raise RuntimeError(f"asynchronous pofa_build step failed its ticket check (status {rc})")
            n = len(used)
            used.clear()
            return n

    if world > 1:
        def check_tickets():
            torch.cuda.synchronize()
            worst = 0
            for tk, guess in sh_used:
                rc = fhv.storage.ticket_status(tk, guess)
                worst = worst or rc
            n = len(sh_used)
            sh_used.clear()
            codes = comm.all_gather_int(worst)  # every rank's tickets (a lower rank's miss moves the bases)
            if any(codes):
                raise RuntimeError(f"speculative sharded build failed its ticket check (statuses {codes})")
            return n
    for _ in range(args.warmup):
        vol = step()
    torch.cuda.synchronize()
    check_tickets()
    n_frags = vol.total if world > 1 else vol.pool.next_free

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- one step captured in a CUDA graph (N = 1, asynchronous steps) ------
    # The whole step -- POFA build (every kernel, memset and copy) + splat --
    # is captured once on its own stream and replayed K times; each replay
    # also checks its build's ticket on the device (sticky status + count).
    graph = None
    acc = torch.zeros(2, dtype=torch.int64, device=dev)

    def make_graph(exact: bool, tris=None, out=None):
        """One step -- POFA build (every kernel, memset and copy) + splat --
        captured on its own stream; each replay also checks its build ticket
        on the device (sticky status + count).  tris / out: the scene and
        image buffers it reads and writes (default: ds / img)."""
        gs = torch.cuda.Stream(dev)
        gticket = torch.zeros(4, dtype=torch.int64).pin_memory()
        g_tris = ds if tris is None else tris
        g_out = img if out is None else out

        def graph_step():
            v = fhv.pofa_build(scene, strat, cfg, L, exact_order=exact, device=dev, tris=g_tris, sync=False,
                               ticket=gticket)
            rc = _lib.load().fhv_ticket_accumulate(_lib.ctx(dev), int(n_frags), _lib.ptr(acc), _lib.stream_ptr(dev))
            _lib.check(rc, "ticket")
            fhv.splat_render(v.pool, view, w["lights"], w["radius"], scene.materials, out=g_out, packed=args.packed,
                             shading=shading)
            return v
        with torch.cuda.stream(gs):
            for _ in range(2):  # this stream's context: speculative item plan, scratch buffers
                graph_step()
        torch.cuda.synchronize()
        acc.zero_()
        g = torch.cuda.CUDAGraph()
        l0 = _lib.launches(dev)
        with torch.cuda.graph(g, stream=gs):
            gv = graph_step()
        n_launch = _lib.launches(dev) - l0
        torch.cuda.synchronize()
        acc.zero_()
        g.replay()  # one untimed replay
        torch.cuda.synchronize()
        return g, gv, n_launch, gs

    def time_graph(g, k):
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        acc.zero_()
        torch.cuda.synchronize()
        ea.record(stream)
        for _ in range(k):
            g.replay()
        eb.record(stream)
        torch.cuda.synchronize()
        bad_, checked_ = (int(x) for x in acc.cpu().tolist())
        if bad_ or checked_ != k:
            raise RuntimeError(f"graph replays: build ticket status {bad_}, {checked_}/{k} checked")
        return ea.elapsed_time(eb) / k

    stream = torch.cuda.current_stream(dev)
    if world == 1 and not args.sync_steps and not args.no_graph:
        graph, gvol, per_replay, gstream = make_graph(args.exact_order)

    # ---- device-resident timed region --------------------------------------
    # (no per-launch events inside it; the per-kernel shares come from a
    # separate profiled pass of the same steps below)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _lib.launches(dev)
    barrier()
    if graph is not None:
        acc.zero_()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                vol = step()
        e1.record(stream)
        barrier()
    if graph is not None:
        bad, checked = (int(x) for x in acc.cpu().tolist())
        if bad or checked != args.steps:
            raise RuntimeError(f"graph replays: build ticket status {bad}, {checked}/{args.steps} checked")
        async_checked = checked
        vol = gvol
        gpu_launches = per_replay * args.steps
    else:
        async_checked = check_tickets()
        gpu_launches = _lib.launches(dev) - launches0
    ms = e0.elapsed_time(e1)
    # what the last timed step produced, for the parity check against the oracle
    shot = None
    if world == 1 and not args.profile_only:
        hp = vol.pool.numpy()
        shot = {"depth": img.depth.cpu().numpy().copy(), "rgba": img.pixels.cpu().numpy().copy(),
                "pool": {k: hp[k].copy() for k in ("position", "normal", "material_id", "object_id",
                                                    "prev_index")},
                "offsets": vol.directory.offsets.cpu().numpy().copy()}
    # per-kernel CUDA events on the launching stream (LaunchScope, fhv_abi.cu)
    _lib.prof_enable(dev, True)
    _lib.prof_collect(dev)  # reset
    barrier()
    ep0, ep1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ep0.record(stream)
    for _ in range(args.steps):
        vol = step()
    ep1.record(stream)
    barrier()
    check_tickets()
    ms_profiled = ep0.elapsed_time(ep1)
    prof = _lib.prof_collect(dev)
    _lib.prof_enable(dev, False)
    # the other in-leaf order, same graph-replay timing (exact <-> fast)
    other = None
    if graph is not None and not args.profile_only:
        g2, _, _, _ = make_graph(not args.exact_order)
        ms2 = time_graph(g2, args.steps)
        other = {"exact_order": not args.exact_order, "ms_per_step": ms2, "value": n_frags / (ms2 / 1e3)}
        del g2
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        t_max = all_max(t_max)
    ms = float(t_max.item())
    ms_step = ms / args.steps
    value = n_frags * args.steps / (ms / 1e3)

    # per-stage shares + roofline of the dominant kernel
    stage_ms = {k: v[0] / args.steps for k, v in prof.items()}
    dominant = max(prof, key=lambda k: prof[k][0])
    T = scene.n_triangles
    P = W * H
    algo_bytes = {  # minimal bytes per launch
        "emit_pofa": 176 * T + 36 * n_frags,
        "count_leaves": 72 * T + 4 * 8 ** L,
        "scan_leaves": 8 * 8 ** L + 8 ** (L - 1),
        "splat_depth": 12 * n_frags + 8 * P,
        "splat_index": 12 * n_frags + 8 * P,
        "splat_resolve": 8 * P + 4 * P + 40 * P,
        "job_setup": (72 + 24 + 80 + 4) * T,
        "leaf_order": 4 * n_frags,  # the ranks read; moved records are the fix-up's own traffic
    }
    peak, peak_kind = peaks()
    roof = None
    if dominant in algo_bytes and world == 1:  # per-kernel bytes below are for the unsharded (N=1) launch
        per_launch_ms = prof[dominant][0] / prof[dominant][1]
        ach = algo_bytes[dominant] / (per_launch_ms / 1e3) / 1e9
        traffic, ncu = None, {}
        tf = os.path.join(ROOT, "profiles", f"ncu_{dominant}.json")
        if os.path.exists(tf):
            try:
                ncu = json.load(open(tf))
                traffic = ncu.get("dram_bytes_per_launch")
            except Exception:
                traffic, ncu = None, {}
        roof = {"bound": "hbm", "kernel": dominant, "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic, "algorithmic_bytes": algo_bytes[dominant],
                "peak_kind": peak_kind, "ms_per_launch": round(per_launch_ms, 4)}
        winst = ncu.get("warp_inst_per_launch")
        if winst:  # the limiter: instruction issue (4 warp instructions / SM / clock)
            mhz = clk.summary().get("sm_mhz") or 1965
            n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
            cap = n_sm * 4 * mhz * 1e6 * per_launch_ms / 1e3
            roof["issue"] = {"warp_inst_per_launch": winst, "peak_warp_inst_per_launch": int(cap),
                             "frac": round(winst / cap, 4),
                             "note": "executed warp instructions from the ncu capture in profiles/ncu_<stage>.json "
                                     "over this run's launch time x SMs x 4 schedulers x SM clock"}
    # atomic / reduction throughput of the atomic-bound stages (north star:
    # "achieved HBM GB/s ... and atomic throughput"): L2 atomic requests per
    # launch from the committed ncu capture (profiles/ncu_<stage>.json) over
    # this run's per-launch time, and the L1 RED / ATOM pipe utilisation ncu saw
    atomics = None
    if world == 1:
        atomics = {}
        for st_name, kind in (("count_leaves", "red"), ("emit_pofa", "atom"), ("splat_depth", "red"),
                              ("splat_index", "red")):
            tf = os.path.join(ROOT, "profiles", f"ncu_{st_name}.json")
            if st_name not in prof or not os.path.exists(tf):
                continue
            try:
                a = json.load(open(tf)).get("atomics") or {}
            except Exception:
                continue
            req = a.get(f"{kind}_requests_l2")
            if not req:
                continue
            per_launch = prof[st_name][0] / prof[st_name][1] / 1e3
            atomics[st_name] = {"op": "RED" if kind == "red" else "ATOM", "l2_requests_per_launch": int(req),
                                "l2_requests_per_s": req / per_launch,
                                "l1_pipe_pct_ncu": a.get(f"{kind}_l1_pipe_pct")}
    capture_ms = sum(v for k, v in stage_ms.items() if not k.startswith("splat"))
    recon_ms = sum(v for k, v in stage_ms.items() if k.startswith("splat"))
    step_bytes = (2 * 176 * T + 36 * n_frags + 12 * 8 ** L + (8 ** L - 1) // 7  # POFA capture
                  + 12 * n_frags + 28 * P + 40 * P)                              # splat + f64 rgba/depth
    # ---- end to end: pinned host scene in, image out ------------------------
    # Every step copies its scene from pinned host memory and reads its f64
    # image + depth back.  The copies run on their own streams, double
    # buffered, so step k+1's upload and step k-1's read-back overlap step
    # k's kernels (a two-deep pipeline, as a serving loop would run it); the
    # step itself is a replay of the captured build + splat of its buffer
    # set (FHV_E2E_GRAPH=0: the plain asynchronous calls, 1.83-1.88 against
    # 1.79-1.81 ms per step).
    if not args.profile_only:
        NB = int(os.environ.get("FHV_E2E_BUFFERS", "2"))  # pipeline depth (scene / image buffer sets)
        # The scene crosses PCIe every step.  --upload indexed (default): as an
        # IndexedMesh (shared vertex rows + u32 faces, 43 MB for C3 instead of
        # the 149-MB triangle soup) that the device expands into the soup
        # arrays, byte for byte (checked below), face normals re-derived with
        # make_triangle's arithmetic.  --upload soup: the triangle arrays as such.
        from paper_2211_15460_b200.device import IndexedMesh, IndexedUpload
        probe = DeviceScene(scene, dev)
        derive_fn = bool(torch.equal(probe.fnrm.clone(), probe.derive_face_normals()))
        indexed = args.upload == "indexed" and derive_fn
        if indexed:
            mesh = IndexedMesh.from_scene(scene)
            arrays = mesh.arrays()
            stage = [IndexedUpload(mesh, dev) for _ in range(NB)]
            for d_, src in zip(stage[0].tensors(), arrays):
                d_.copy_(torch.from_numpy(np.ascontiguousarray(src)))
            ref_soup = DeviceScene(scene, dev)
            probe.pos.zero_(); probe.vnrm.zero_(); probe.fnrm.zero_()
            probe.load_indexed(stage[0])
            idx_ok = all(torch.equal(getattr(probe, f).view(torch.int64) if getattr(probe, f).dtype == torch.float64
                                     else getattr(probe, f), getattr(ref_soup, f).view(torch.int64)
                                     if getattr(ref_soup, f).dtype == torch.float64 else getattr(ref_soup, f))
                         for f in ("pos", "vnrm", "fnrm", "mat", "obj"))
            if not idx_ok:
                raise RuntimeError("indexed expansion differs from the triangle arrays")
            del ref_soup
        else:
            arrays = (scene.positions, scene.normals) + (() if derive_fn else (scene.face_normals,)) + \
                (scene.material_id.view(np.int32), scene.object_id.view(np.int32))
        del probe
        pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in arrays]
        bufs_in = [ds] + [DeviceScene(scene, dev) for _ in range(NB - 1)]
        bufs_out = [img] + [ImageBuffer(W, H, torch.empty((H, W, 4), dtype=torch.float64, device=dev),
                                        torch.empty((H, W), dtype=torch.float64, device=dev)) for _ in range(NB - 1)]
        out_px = [torch.empty((H, W, 4), dtype=torch.float64).pin_memory() for _ in range(NB)]
        out_dp = [torch.empty((H, W), dtype=torch.float64).pin_memory() for _ in range(NB)]
        h2d = sum(p.numel() * p.element_size() for p in pin)

        def dst_of(k):
            if indexed:
                return stage[k % NB].tensors()
            b = bufs_in[k % NB]
            return (b.pos, b.vnrm) + (() if derive_fn else (b.fnrm,)) + (b.mat.view(torch.int32), b.obj.view(torch.int32))
        # the link itself: the same pinned uploads alone (PCIe bound of the e2e line)
        torch.cuda.synchronize()
        el0, el1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        el0.record(stream)
        for _ in range(3):
            for d_, src in zip(dst_of(0), pin):
                d_.copy_(src, non_blocking=True)
        el1.record(stream)
        torch.cuda.synchronize()
        h2d_gbs = 3 * h2d / (el0.elapsed_time(el1) / 1e3) / 1e9
        d2h = out_px[0].numel() * 8 + out_dp[0].numel() * 8
        # steps: the build + splat as CUDA-graph replays, one graph per buffer
        # set (as in the device-resident loop; no host-side allocation that
        # could serialise the pipeline), else the plain asynchronous calls
        e2e_graphs = None
        if graph is not None and os.environ.get("FHV_E2E_GRAPH", "1") != "0":
            e2e_graphs = [make_graph(args.exact_order, bufs_in[i], bufs_out[i])[0] for i in range(NB)]
            torch.cuda.synchronize()
            acc.zero_()
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        K = args.steps
        ev = lambda: torch.cuda.Event()  # noqa: E731
        e_in, e_done, e_out = [ev() for _ in range(K)], [ev() for _ in range(K)], [ev() for _ in range(K)]
        e_start = ev()

        def upload(k):
            s_in.wait_event(e_start)
            if k >= NB:
                s_in.wait_event(e_done[k - NB])  # buffer k%NB free again
            with torch.cuda.stream(s_in):
                for d, src in zip(dst_of(k), pin):
                    d.copy_(src, non_blocking=True)
                e_in[k].record(s_in)

        def readback(k):
            s_out.wait_event(e_done[k])
            with torch.cuda.stream(s_out):
                out_px[k % NB].copy_(bufs_out[k % NB].pixels, non_blocking=True)
                out_dp[k % NB].copy_(bufs_out[k % NB].depth, non_blocking=True)
                e_out[k].record(s_out)

        barrier()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        e_start.record(stream)
        upload(0)
        for k in range(K):
            if k + 1 < K:
                upload(k + 1)
            stream.wait_event(e_in[k])
            if k >= NB:
                stream.wait_event(e_out[k - NB])  # image buffer k%NB read back
            if indexed:
                bufs_in[k % NB].load_indexed(stage[k % NB])  # gather + ids + face normals, on the device
            elif derive_fn:
                bufs_in[k % NB].derive_face_normals()
            if e2e_graphs is not None:
                e2e_graphs[k % NB].replay()
            else:
                step(bufs_in[k % NB], bufs_out[k % NB])
            e_done[k].record(stream)
            readback(k)
        for k in range(max(0, K - NB), K):
            stream.wait_event(e_out[k])
        e3.record(stream)
        barrier()
        check_tickets()
        if e2e_graphs is not None:
            bad_e, checked_e = (int(x) for x in acc.cpu().tolist())
            if bad_e or checked_e != K:
                raise RuntimeError(f"e2e graph replays: build ticket status {bad_e}, {checked_e}/{K} checked")
        ms_e2e = e2.elapsed_time(e3)
        t2 = torch.tensor([ms_e2e], dtype=torch.float64, device=dev)
        if world > 1:
            t2 = all_max(t2)
        ms_e2e = float(t2.item())
        torch.cuda.synchronize()
        ok = np.array_equal(out_dp[(K - 1) % NB].numpy(), bufs_out[(K - 1) % NB].depth.cpu().numpy())
        e2e = {"value": n_frags * args.steps / (ms_e2e / 1e3), "unit": "frag/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e / args.steps,
               "pipeline": f"{NB} buffers: H2D(k+1) and D2H(k-1) on copy streams overlap step k",
               "steps": ("CUDA-graph replays of the captured build + splat (one graph per buffer set; every build "
                         "ticket checked on the device)" if e2e_graphs is not None else "asynchronous API calls"),
               "upload": ("indexed mesh: %d shared vertex rows + %d u32 faces, expanded on the device into the "
                          "triangle arrays (checked byte-identical before timing)" % (mesh.n_vertices, mesh.n_triangles)
                          if indexed else "triangle arrays"),
               "face_normals": "derived on device (bit-identical)" if derive_fn else "uploaded",
               "readback_matches_device": bool(ok), "h2d_link_gbs": round(h2d_gbs, 1)}
    else:
        e2e = None

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.profile_only:
        import numpy as np
        nt = host_threads()
        # threads=1: the reference's sequential (canonical) order -- a threaded
        # oracle run keeps counts / offsets / image but not the in-leaf order
        n, tc, ts, (rv, rrgba, rdepth) = cpu_run(w, 1, keep=True)
        single = (n, tc, ts)
        parity = {"vs": "oracle port (oracle/fhv_oracle.c, pinned to the reference's golden vectors) on the same "
                        "inputs: the last timed step's image and pool",
                  "fragments_equal": int(n) == int(n_frags),
                  "offsets_bit_exact": bool(np.array_equal(shot["offsets"], rv["offsets"])),
                  "depth_bit_exact": bool(np.array_equal(shot["depth"], rdepth)),
                  "rgba_max_abs_err": float(np.max(np.abs(shot["rgba"] - rrgba))),
                  "rgba_tol": 1e-12}
        if args.exact_order:
            parity["pool_bit_exact"] = all(np.array_equal(shot["pool"][k], rv["pool"][k]) for k in shot["pool"])
        else:
            parity["pool"] = "fast order: per-leaf multiset (records not compared)"
        parity["ok"] = bool(parity["fragments_equal"] and parity["offsets_bit_exact"] and parity["depth_bit_exact"]
                            and parity["rgba_max_abs_err"] <= 1e-12 and parity.get("pool_bit_exact", True))
        del rv, rrgba, rdepth
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile_only:
        nt = host_threads()
        cpu_run(w, nt)  # warm-up (page faults, thread start)
        n, tc, ts = cpu_run(w, nt)
        n1, tc1, ts1 = single if parity is not None else cpu_run(w, 1)
        cpu = {"value": n / (tc + ts), "unit": "frag/s", "cores": nt, "kind": "port",
               "sample": f"one full C3 step on the host (oracle/fhv_oracle.c, {nt} threads): capture {tc:.2f} s + "
                         f"splat {ts:.2f} s",
               "capture_s": tc, "splat_s": ts,
               "single_thread": {"value": n1 / (tc1 + ts1), "capture_s": tc1, "splat_s": ts1}}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "frag/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded icosphere field, no dataset)",
                "config": CONFIG,  # the workload; identical to the reference arm's
                "run": dict(fragments=n_frags,
                               parallelism=(f"morton-range shards x{world} ({os.environ.get('FHV_BENCH_BACKEND', 'nccl')})"
                                            if world > 1 else "single"),
                               composite=composite if world > 1 else None,
                               exact_order=bool(args.exact_order), splat="packed" if args.packed else "exact",
                               host=("CUDA-graph replays of one captured asynchronous step (POFA build + splat, "
                                     "every kernel / memset / copy re-executed), all %d build tickets checked on the "
                                     "device" % async_checked) if graph is not None else
                               ("asynchronous steps: %s, all %d tickets verified after the timed loop%s"
                                % ("pofa_build_shard(sync=False) (no host wait, no collective in the build)"
                                   if world > 1 else "pofa_build(sync=False)", async_checked,
                                   " (every rank's)" if world > 1 else "")
                                if async_checked else "synchronous steps")),
                "novel_view_fps": 1e3 / recon_ms if recon_ms else None,
                "capture_frag_per_s": n_frags / (capture_ms / 1e3) if capture_ms else None,
                "step_gbs": step_bytes / (ms_step / 1e3) / 1e9, "step_bytes": step_bytes,
                "stage_ms": {k: round(v, 4) for k, v in sorted(stage_ms.items(), key=lambda kv: -kv[1])},
                "gap_ms_per_step": round(ms_profiled / args.steps - sum(stage_ms.values()), 4),
                "ms_per_step_profiled": round(ms_profiled / args.steps, 4),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches,
                "parity": parity, "other_order": other, "atomics": atomics,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
