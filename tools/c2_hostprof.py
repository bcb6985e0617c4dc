#!/usr/bin/env python
"""Host-side view of the C2 step (POFL build + 1080p ray cast): enqueue vs
wall time per step, the synced build alone, and a cProfile of the step.
build_pofl waits for its fragment total, so each step's capture also waits
for the previous step's ray cast -- the gap between the kernels' sum and the
measured C2 ms_per_step.

    python tools/c2_hostprof.py
"""
import time, cProfile, pstats, sys
sys.path.insert(0, '.')
import torch, bench
import paper_2211_15460_b200 as fhv
from paper_2211_15460_b200 import sample_scenes
from paper_2211_15460_b200.raster import CaptureStrategy, RasterConfig
from paper_2211_15460_b200.scene import capture_camera, viewpoint_camera
from paper_2211_15460_b200.lights import headlight
from paper_2211_15460_b200.device import DeviceShading, device_scene
dev = torch.device("cuda", 0)
scene = sample_scenes.spheres100k(); ns = CaptureStrategy.normal_space()
cam = capture_camera(scene, "+z", 1080)
cfg = RasterConfig((1920, 1080), RasterConfig.from_camera(cam).projection, extent=1.0)
view = viewpoint_camera("+x", (1920, 1080), "perspective"); lights = [headlight(view)]
sh = DeviceShading(scene.materials, lights, dev)
vol0 = fhv.build_pofl(scene, ns, cfg, 8, device=dev); rcfg = fhv.default_raycast_config(vol0)
buf = fhv.ImageBuffer(1920, 1080, torch.zeros((1080, 1920, 4), dtype=torch.float64, device=dev), torch.zeros((1080, 1920), dtype=torch.float64, device=dev))
def step():
    vol = fhv.build_pofl(scene, ns, cfg, 8, device=dev)
    buf.pixels.zero_()
    fhv.render_raycast(vol, view, lights, rcfg, out=buf, sync=False, shading=sh)
    return vol
for _ in range(5): step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20): v = step()
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"enqueue {1e3*(t1-t0)/20:.3f} ms/step, wall {1e3*(t2-t0)/20:.3f} ms/step")
tb = 0.0
for _ in range(10):
    torch.cuda.synchronize(); a = time.perf_counter(); v = fhv.build_pofl(scene, ns, cfg, 8, device=dev); torch.cuda.synchronize(); tb += time.perf_counter() - a
print(f"build_pofl alone (synced) {1e3*tb/10:.3f} ms")
pr = cProfile.Profile(); pr.enable()
for _ in range(10): step()
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
