"""C2 / C5-view ray-cast probe: stage times of the packet and hand-off kernels,
rays handed off, RaycastStats, and (with --check) the image against the
per-ray-only library build given as FHV_LIB_REF.

    python tools/ray_probe.py [--reps N] [--c5]
"""
from __future__ import annotations

import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2211_15460_b200 as fhv  # noqa: E402
from paper_2211_15460_b200 import _lib, sample_scenes  # noqa: E402
from paper_2211_15460_b200.lights import headlight  # noqa: E402
from paper_2211_15460_b200.raster import CaptureStrategy, RasterConfig  # noqa: E402
from paper_2211_15460_b200.scene import capture_camera, viewpoint_camera  # noqa: E402


def main():
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
    dev = torch.device("cuda:0")
    ns = CaptureStrategy.normal_space()
    if "--c5" in sys.argv:
        scene = sample_scenes.scatter1m()
        cam = capture_camera(scene, "+z", 1080)
        cfg = RasterConfig((1920, 1080), RasterConfig.from_camera(cam).projection, extent=1.0)
        vol = fhv.pofa_build(scene, ns, cfg, 8, device=dev)
        views = sample_scenes.c5_views(64)[:4]
    else:
        scene = sample_scenes.spheres100k()
        cam = capture_camera(scene, "+z", 1080)
        cfg = RasterConfig((1920, 1080), RasterConfig.from_camera(cam).projection, extent=1.0)
        vol = fhv.build_pofl(scene, ns, cfg, 8, device=dev)
        views = [viewpoint_camera("+x", (1920, 1080), "perspective")]
    rcfg = fhv.default_raycast_config(vol)
    for mode in ("transparency", "opaque_nearest"):
        rc = dataclasses.replace(rcfg, mode=mode)
        for vi, view in enumerate(views):
            lights = [headlight(view)]
            img, st = fhv.render_raycast(vol, view, lights, rc)
            torch.cuda.synchronize()
            hand = _lib.raycast_diag(dev)
            _lib.prof_enable(dev, True)
            _lib.prof_collect(dev)
            for _ in range(reps):
                fhv.render_raycast(vol, view, lights, rc, sync=False)
            torch.cuda.synchronize()
            prof = _lib.prof_collect(dev)
            _lib.prof_enable(dev, False)
            ms = {k: round(v[0] / reps, 4) for k, v in prof.items() if v[0] > 0}
            print(f"mode={mode} view={vi} handoffs={hand} stats={st.as_dict()} ms={ms}", flush=True)


if __name__ == "__main__":
    main()
