"""North-star facade: ``capture(scene, variant=...)`` and ``reconstruct(fhv, view)``.

Thin dispatch onto the reference-named builders (build_ppfl / build_pofl /
pofa_build) and reconstructions (splat_render / render_raycast).
"""
from __future__ import annotations

from .lights import headlight
from .raster import CaptureStrategy, RasterConfig
from .raycast import RaycastConfig, default_raycast_config, render_raycast
from .render import splat_render
from .scene import capture_camera
from .storage import build_pofl, build_ppfl, pofa_build

__all__ = ["capture", "reconstruct"]


def capture(scene, variant: str = "POFA", resolution=(1920, 1080), levels: int = 8, strategy=None,
            capacity=None, overalloc: float = 10.0, exact_order: bool | None = None, device=None):
    """Capture a scene into an FHV store.  ``variant`` in {PPFL, POFL, POFA};
    ``resolution`` is the RasterConfig resolution (the capture grid is
    resolution[1]^2, fhv/raster.py:359).  ``exact_order`` defaults to each
    builder's own default (POFA: the reference's exact order)."""
    order = {} if exact_order is None else {"exact_order": exact_order}
    variant = variant.upper()
    cam = capture_camera(scene, "+z", int(resolution[1]))
    cfg = RasterConfig(tuple(resolution), RasterConfig.from_camera(cam).projection, extent=1.0)
    if variant == "PPFL":
        return build_ppfl(scene, cfg, strategy or CaptureStrategy.one_view(), capacity, overalloc, device=device,
                          **order)
    strategy = strategy or CaptureStrategy.normal_space()
    if variant == "POFL":
        return build_pofl(scene, strategy, cfg, levels, capacity, overalloc, device=device, **order)
    if variant == "POFA":
        return pofa_build(scene, strategy, cfg, levels, device=device, **order)
    raise ValueError(f"unknown variant {variant!r}")


def reconstruct(fhv, view, method: str = "splat", lights=None, radius: float | None = None, mode: str = "transparency",
                background=(0.0, 0.0, 0.0, 0.0), materials=None, packed: bool = False, collect_ids: bool = False):
    """Reconstruct one novel view (a Camera).  ``method``: splat | raycast."""
    lights = lights if lights is not None else [headlight(view)]
    materials = materials if materials is not None else fhv.materials
    if method == "splat":
        r = radius if radius is not None else 1.0 / fhv.capture_resolution
        return splat_render(fhv.pool, view, lights, r, materials, background, packed=packed)
    if method == "raycast":
        cfg = default_raycast_config(fhv, mode=mode) if radius is None else RaycastConfig(radius, 1.0, mode, 2.0 * radius)
        return render_raycast(fhv, view, lights, cfg, materials, background, collect_ids=collect_ids)
    raise ValueError(f"unknown method {method!r}")
