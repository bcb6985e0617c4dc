#!/usr/bin/env python
"""Host-side profile of the bench step (C3): where the wall time of a step goes
between Python, the C-ABI calls (which include their internal syncs) and the
GPU.  python tools/host_profile.py [steps]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(steps=20):
    import torch
    import bench
    import paper_2211_15460_b200 as fhv
    from paper_2211_15460_b200.device import DeviceShading, device_scene
    from paper_2211_15460_b200.lights import ImageBuffer
    dev = torch.device("cuda", 0)
    w = bench.workload()
    scene, cfg, strat, L, view = w["scene"], w["cfg"], w["strategy"], w["levels"], w["view"]
    ds = device_scene(scene, dev)
    shading = DeviceShading(scene.materials, w["lights"], dev)
    W, H = view.resolution
    img = ImageBuffer(W, H, torch.empty((H, W, 4), dtype=torch.float64, device=dev),
                      torch.empty((H, W), dtype=torch.float64, device=dev))

    asynchronous = os.environ.get("HOSTPROF_ASYNC", "1") != "0"
    tickets = torch.zeros((4 * (steps + 8), 4), dtype=torch.int64).pin_memory()
    used = [0]

    def step():
        tk = tickets[used[0] % len(tickets)]
        used[0] += 1
        vol = fhv.pofa_build(scene, strat, cfg, L, device=dev, tris=ds, sync=not asynchronous, ticket=tk)
        fhv.splat_render(vol.pool, view, w["lights"], w["radius"], scene.materials, out=img, shading=shading)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{'asynchronous' if asynchronous else 'synchronous'} steps: host enqueue per step "
          f"{1e3 * (t1 - t0) / steps:.3f} ms, wall per step {1e3 * (time.perf_counter() - t0) / steps:.3f} ms")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
    # time inside each C-ABI call (includes the library's own syncs) vs the rest
    from paper_2211_15460_b200 import _lib
    lib = _lib.load()
    acc = {}

    class Timed:
        def __init__(self, name, fn):
            self.name, self.fn = name, fn

        def __call__(self, *a):
            t = time.perf_counter()
            r = self.fn(*a)
            acc[self.name] = acc.get(self.name, 0.0) + time.perf_counter() - t
            return r
    for name in ("fhv_pofa_build", "fhv_splat"):
        setattr(lib, name, Timed(name, getattr(lib, name)))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps
    print(f"wall per step {1e3 * wall:.3f} ms; inside C calls per step: " +
          ", ".join(f"{k} {1e3 * v / steps:.3f} ms" for k, v in acc.items()) +
          f"; python outside {1e3 * (wall - sum(acc.values()) / steps):.3f} ms")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 20)
