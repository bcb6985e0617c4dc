"""Time the SHIPPED reference (``fhv``, /root/reference) on a prefix of the C3
workload, both backends, threads=1 -- context for bench.py's cpu_baseline
(VERDICT r01 "a timing of the shipped reference itself").

The reference cannot travel to the GPU box (/root/reference is absent there),
so this runs in the build container and writes profiles/r02_shipped_reference.json;
bench.py quotes it beside the oracle-port baseline it measures on the box.

  * scene: the first ``--tris`` triangles of scatter1M (the reference-pinned
    scene, tests/test_scene_pinning.py), as reference ``Triangle`` objects;
  * capture: ``pofa_build(scene, NormalSpace, cfg 1920x1080 ortho extent 1,
    L=8, threads=1)``, timed, then scaled linearly to 983,040 triangles;
  * splat: ``splat_render`` of that prefix's pool at 1920x1080, r = 1/1080,
    scaled by fragments (the splat is linear in the pool);
  * backends: "python" (NumPy kernels, as shipped) and "compiled" (Cython
    kernels with the 5 pointer casts of SURVEY.md Appendix C).

Usage: python tools/time_shipped_reference.py [--tris 100000]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_backend(compiled: bool, n_tris: int) -> dict:
    code = f"""
import json, sys, time, os
sys.path.insert(0, {os.path.join(ROOT, 'tests', 'golden')!r})
sys.path.insert(0, {ROOT!r})
import numpy as np
from make_golden import prepare_reference
prepare_reference(compiled={compiled})
import fhv
from fhv import _backend
from fhv.scene import Scene, Material, make_triangle, capture_camera, viewpoint_camera
from fhv.raster import RasterConfig, CaptureStrategy
from fhv.storage import pofa_build
from fhv.render import splat_render, headlight
from paper_2211_15460_b200 import sample_scenes
s = sample_scenes.scatter1m()
n = {n_tris}
tris = []
for t in range(n):
    P, N = s.positions[t], s.normals[t]
    tr = make_triangle(P[0], P[1], P[2], N[0], N[1], N[2], int(s.material_id[t]), int(s.object_id[t]))
    tris.append(tr)
mats = [Material(m.diffuse, m.specular, m.shininess, m.alpha) for m in s.materials]
scene = Scene.from_triangles(tris, mats)
cam = capture_camera(scene, "+z", 1080)
cfg = RasterConfig((1920, 1080), RasterConfig.from_camera(cam).projection, extent=1.0)
t0 = time.perf_counter()
vol = pofa_build(scene, CaptureStrategy.normal_space(), cfg, 8, threads=1)
t1 = time.perf_counter()
view = viewpoint_camera("+x", (1920, 1080), "perspective")
img = splat_render(vol.pool, view, [headlight(view)], 1.0 / 1080, scene.materials)
t2 = time.perf_counter()
print(json.dumps({{"backend": _backend.active_backend() if hasattr(_backend, "active_backend") else str(_backend),
                  "tris": n, "fragments": int(vol.pool.next_free), "capture_s": t1 - t0, "splat_s": t2 - t1}}))
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tris", type=int, default=100_000)
    args = ap.parse_args()
    T_FULL, N_FULL = 983_040, 4_558_046  # C3 triangles / fragments (bench.py)
    res = {"what": "shipped reference fhv (/root/reference) on a prefix of the C3 workload, threads=1, "
                   "scaled linearly to the full C3 step (capture by triangles, splat by fragments)",
           "host": platform.processor() or platform.machine(), "cpu_count": os.cpu_count(), "runs": []}
    for compiled in (True, False):
        r = run_backend(compiled, args.tris)
        cap_full = r["capture_s"] * T_FULL / r["tris"]
        spl_full = r["splat_s"] * N_FULL / max(1, r["fragments"])
        r.update({"compiled": compiled, "capture_s_scaled": cap_full, "splat_s_scaled": spl_full,
                  "frag_per_s": N_FULL / (cap_full + spl_full)})
        res["runs"].append(r)
        print(json.dumps(r), flush=True)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(res, open(os.path.join(ROOT, "profiles", "r02_shipped_reference.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
