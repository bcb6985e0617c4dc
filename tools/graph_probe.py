#!/usr/bin/env python
"""Experiment: one C3 step (asynchronous POFA build + splat) captured in a
CUDA graph and replayed, vs the same step enqueued from Python each time.

    python tools/graph_probe.py [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(steps=50):
    import numpy as np
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
    tk = torch.zeros(4, dtype=torch.int64).pin_memory()

    def step():
        vol = fhv.pofa_build(scene, strat, cfg, L, device=dev, tris=ds, sync=False, ticket=tk)
        fhv.splat_render(vol.pool, view, w["lights"], w["radius"], scene.materials, out=img, shading=shading)
        return vol

    gs = torch.cuda.Stream(dev)
    with torch.cuda.stream(gs):
        fhv.pofa_build(scene, strat, cfg, L, device=dev, tris=ds)  # the exact total (pool size guess)
        for _ in range(3):
            step()
    gs.synchronize()
    ref = img.pixels.clone()

    def timed(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(gs):
            torch.cuda.synchronize()
            e0.record(gs)
            for _ in range(steps):
                fn()
            e1.record(gs)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    t_loop = timed(step)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        step()
    torch.cuda.synchronize()
    t_graph = timed(g.replay)
    guesses = list(ds._pofa_totals.values())
    tick = [int(fhv._lib.load().fhv_ticket_check(fhv.storage.c_vp_of(tk), int(gv))) for gv in guesses]
    diff = (img.pixels - ref).abs()
    print(f"python loop {t_loop:.4f} ms/step, graph replay {t_graph:.4f} ms/step; ticket status {tick} "
          f"(guesses {guesses}, ticket {tk.tolist()}); image max diff {float(diff.max()):.3g} on "
          f"{int((diff.amax(-1) > 0).sum())} pixels (atomic in-leaf order -> depth ties may pick another winner)")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 50)
