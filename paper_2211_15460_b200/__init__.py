"""B200-native fragment-history volumes (arXiv 2211.15460).

Drop-in for the reference package ``fhv`` on its hot path: capture a triangle
scene into PPFL / POFL / POFA fragment stores with a CUDA software rasteriser,
then reconstruct novel views by point splatting or octree ray casting -- all
in hand-written sm_100a kernels behind a C ABI (include/fhv_b200.h).
"""
from . import kernels, sample_scenes
from .api import capture, reconstruct
from .ingest import load_material_table, load_scene, save_material_table, save_scene
from .capture import capture_fragments, capture_pass
from .lights import (GBuffer, ImageBuffer, Light, composite_over, front_to_back_accumulate, headlight,
                     write_float_dump, write_ppm)
from .raster import (CaptureStats, CaptureStrategy, EmittedFragment, FragmentBatch, ListSink, RasterConfig,
                     capture_plan, ortho_projection, perspective_projection, rasterize_triangle, rasterize_triangles,
                     tangent_basis, world_pixel_footprint)
from .raycast import (HitRecord, Ray, RaycastConfig, RaycastStats, default_raycast_config, gather_ray_hits,
                      gen_primary_ray, intersect_fragment, primary_rays, raycast_pixel, render_raycast,
                      shadow_transmittance, traverse_octree)
from .render import deferred_baseline, project_points, shade, shade_many, splat_render
from .scene import (Aabb, Camera, Material, Scene, SceneError, SceneLoadError, SceneTransform, Triangle, Vertex,
                    capture_camera,
                    make_quad, make_triangle, normalize_scene, viewpoint_camera)
from .storage import (CountingSink, FhvError, FhvPofa, FhvPofl, FhvPpfl, FragmentPool, FragmentRecord,
                      OccupancyPyramid, PofaBuildError, PofaWriteSink, PoflSink, PpflSink, build_pofl, build_ppfl,
                      cell_of, chain_indices, load_snapshot, memory_report, morton_decode, morton_encode, pofa_build,
                      pofl_insert, ppfl_insert, rebuild_pofl_as_pofa, save_snapshot, snapshot_bytes)

__version__ = "0.1.0"
BACKEND_NAME = "b200"
# the reference's flag for "the compiled kernel module imported"; here the
# CUDA library is the only backend (no NumPy fallback), so it is always True
HAVE_COMPILED = True


def active_backend() -> str:
    """The reference reports "compiled" / "python"; this package has exactly one backend."""
    return BACKEND_NAME
