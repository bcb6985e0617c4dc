"""B200-native fragment-history volumes (arXiv 2211.15460).

Drop-in for the reference package ``fhv`` on its hot path: capture a triangle
scene into PPFL / POFL / POFA fragment stores with a CUDA software rasteriser,
then reconstruct novel views by point splatting or octree ray casting -- all
in hand-written sm_100a kernels behind a C ABI (include/fhv_b200.h).
"""
from . import sample_scenes
from .api import capture, reconstruct
from .ingest import load_material_table, load_scene, save_material_table, save_scene
from .capture import capture_fragments, capture_pass
from .lights import (GBuffer, ImageBuffer, Light, composite_over, front_to_back_accumulate, headlight,
                     write_float_dump, write_ppm)
from .raster import (CaptureStats, CaptureStrategy, FragmentBatch, RasterConfig, capture_plan, ortho_projection,
                     perspective_projection, tangent_basis, world_pixel_footprint)
from .raycast import RaycastConfig, RaycastStats, default_raycast_config, primary_rays, render_raycast
from .render import deferred_baseline, splat_render
from .scene import (Aabb, Camera, Material, Scene, SceneError, SceneLoadError, SceneTransform, Triangle, Vertex,
                    capture_camera,
                    make_quad, make_triangle, normalize_scene, viewpoint_camera)
from .storage import (FhvError, FhvPofa, FhvPofl, FhvPpfl, FragmentPool, FragmentRecord, OccupancyPyramid,
                      PofaBuildError, build_pofl, build_ppfl, cell_of, load_snapshot, memory_report, morton_decode,
                      morton_encode, pofa_build, rebuild_pofl_as_pofa, save_snapshot, snapshot_bytes)

__version__ = "0.1.0"
BACKEND_NAME = "b200"


def active_backend() -> str:
    """The reference reports "compiled" / "python"; this package has exactly one backend."""
    return BACKEND_NAME
