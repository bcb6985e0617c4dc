"""Built-in scenes: the reference's fixtures plus the bench workloads.

The four built-ins (``three-quads``, ``icosphere``, ``edge-plane``,
``cornell``) reproduce ``fhv/sample_scenes.py:20-171`` bit for bit (same
vertex lists, same IEEE operations), so their captures can be compared with
golden vectors taken from the reference.  The bench scenes (SURVEY.md
section 8(d), configs C1-C5) are defined here; the large ones are built
struct-of-arrays instead of one ``make_triangle`` call per triangle, with the
same arithmetic (``np.vecdot`` reproduces the BLAS ddot norm used by
``make_triangle``): byte-identical to the same fields built by the
reference's own ``icosphere`` / ``make_triangle`` (tests/test_scene_pinning.py
against tests/golden/scenes_big.json).
"""
from __future__ import annotations

import math

import numpy as np

from .scene import Material, Scene, make_quad, make_triangle

__all__ = ["builtin_names", "builtin_scene", "cornell_box", "cube972", "edge_plane", "icosphere",
           "icosphere_mesh", "layers80", "overlap_quads", "sphere_field", "spheres100k",
           "scatter1m", "unit_quad"]


def unit_quad(z: float = 0.5, alpha: float = 1.0) -> Scene:
    mat = Material(diffuse=(0.8, 0.8, 0.8), alpha=alpha)
    return Scene.from_triangles(make_quad((0, 0, z), (1, 0, z), (1, 1, z), (0, 1, z)), [mat])


def overlap_quads() -> Scene:
    """Paper Fig. 2: three alpha-1/3 quads; inserted green, red, blue; seen
    from +z the depth order is red, green, blue (fhv/sample_scenes.py:27-46)."""
    mats = [Material(diffuse=(0.0, 1.0, 0.0), alpha=1.0 / 3.0),
            Material(diffuse=(1.0, 0.0, 0.0), alpha=1.0 / 3.0),
            Material(diffuse=(0.0, 0.0, 1.0), alpha=1.0 / 3.0)]
    tris = []
    for (x0, x1, y0, y1, z), k in zip(((0.25, 0.75, 0.25, 0.75, 0.5), (0.15, 0.65, 0.35, 0.85, 0.8),
                                        (0.35, 0.85, 0.15, 0.65, 0.2)), range(3)):
        tris += make_quad((x0, y0, z), (x1, y0, z), (x1, y1, z), (x0, y1, z), material_id=k, object_id=k)
    return Scene.from_triangles(tris, mats)


_ICO_BASE_FACES = (
    (0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
    (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
    (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
    (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1),
)


def icosphere_mesh(subdivisions: int):
    """Unit icosphere (vertex list, face list), subdivided by edge midpoints
    re-projected to the sphere; vertex numbering follows the reference."""
    g = (1.0 + math.sqrt(5.0)) / 2.0
    raw = [(-1, g, 0), (1, g, 0), (-1, -g, 0), (1, -g, 0), (0, -1, g), (0, 1, g), (0, -1, -g),
           (0, 1, -g), (g, 0, -1), (g, 0, 1), (-g, 0, -1), (-g, 0, 1)]
    verts = [np.array(v, dtype=np.float64) / np.linalg.norm(v) for v in raw]
    faces = list(_ICO_BASE_FACES)
    for _ in range(subdivisions):
        mid: dict = {}

        def midpoint(a: int, b: int) -> int:
            key = (min(a, b), max(a, b))
            k = mid.get(key)
            if k is None:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                k = mid[key] = len(verts) - 1
            return k

        nxt = []
        for a, b, c in faces:
            ab = midpoint(a, b)
            ca = midpoint(c, a)
            bc = midpoint(b, c)
            nxt += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nxt
    return verts, faces


def icosphere(subdivisions: int = 2, radius: float = 0.35, center=(0.5, 0.5, 0.5),
              alpha: float = 1.0) -> Scene:
    """Opaque icosphere with radial vertex normals (fhv/sample_scenes.py:49-89)."""
    verts, faces = icosphere_mesh(subdivisions)
    center = np.asarray(center, dtype=np.float64)
    mat = Material(diffuse=(0.75, 0.75, 0.78), specular=(0.3, 0.3, 0.3), shininess=32.0, alpha=alpha)
    tris = [make_triangle(center + radius * verts[a], center + radius * verts[b],
                          center + radius * verts[c], verts[a], verts[b], verts[c])
            for a, b, c in faces]
    return Scene.from_triangles(tris, [mat])


def edge_plane(tilt: float = 0.025) -> Scene:
    """Plane nearly parallel to the +z capture axis (fhv/sample_scenes.py:92-106)."""
    def x_at(z):
        return 0.5 - tilt / 2.0 + tilt * (z - 0.1) / 0.8
    mat = Material(diffuse=(0.9, 0.7, 0.2), alpha=1.0)
    return Scene.from_triangles(make_quad((x_at(0.1), 0.1, 0.1), (x_at(0.1), 0.9, 0.1),
                                          (x_at(0.9), 0.9, 0.9), (x_at(0.9), 0.1, 0.9)), [mat])


def cornell_box() -> Scene:
    """Five walls and two boxes, 7 objects, 4 materials (fhv/sample_scenes.py:109-150)."""
    mats = [Material(diffuse=(0.85, 0.85, 0.85)), Material(diffuse=(0.8, 0.15, 0.15)),
            Material(diffuse=(0.15, 0.8, 0.15)),
            Material(diffuse=(0.6, 0.6, 0.65), specular=(0.2, 0.2, 0.2))]
    lo, hi = 0.05, 0.95
    walls = [
        (((lo, lo, lo), (hi, lo, lo), (hi, lo, hi), (lo, lo, hi)), 0, 0),
        (((lo, hi, lo), (lo, hi, hi), (hi, hi, hi), (hi, hi, lo)), 0, 1),
        (((lo, lo, lo), (lo, hi, lo), (hi, hi, lo), (hi, lo, lo)), 0, 2),
        (((lo, lo, lo), (lo, lo, hi), (lo, hi, hi), (lo, hi, lo)), 1, 3),
        (((hi, lo, lo), (hi, hi, lo), (hi, hi, hi), (hi, lo, hi)), 2, 4),
    ]
    tris = []
    for q, m, o in walls:
        tris += make_quad(*q, material_id=m, object_id=o)

    def box(x0, x1, y0, y1, z0, z1, obj):
        faces = [((x0, y0, z1), (x1, y0, z1), (x1, y1, z1), (x0, y1, z1)),
                 ((x1, y0, z0), (x0, y0, z0), (x0, y1, z0), (x1, y1, z0)),
                 ((x0, y0, z0), (x0, y0, z1), (x0, y1, z1), (x0, y1, z0)),
                 ((x1, y0, z1), (x1, y0, z0), (x1, y1, z0), (x1, y1, z1)),
                 ((x0, y1, z1), (x1, y1, z1), (x1, y1, z0), (x0, y1, z0)),
                 ((x0, y0, z0), (x1, y0, z0), (x1, y0, z1), (x0, y0, z1))]
        out = []
        for f in faces:
            out += make_quad(*f, material_id=3, object_id=obj)
        return out

    tris += box(0.15, 0.45, lo, 0.55, 0.15, 0.45, 5)
    tris += box(0.55, 0.85, lo, 0.35, 0.45, 0.75, 6)
    return Scene.from_triangles(tris, mats)


_BUILTIN = {"three-quads": overlap_quads, "icosphere": icosphere, "edge-plane": edge_plane,
            "cornell": cornell_box}


def builtin_names() -> list:
    return sorted(_BUILTIN)


def builtin_scene(name: str) -> Scene:
    try:
        return _BUILTIN[name]()
    except KeyError:
        raise ValueError(f"unknown builtin scene {name!r}; available: {', '.join(builtin_names())}") from None


# ---------------------------------------------------------------------------
# Bench workloads


def cube972() -> Scene:
    """C1: cube [0.1,0.9]^3, 9x9 quads per face, 2 triangles each (972),
    outward winding, one object id per face, one material."""
    mat = Material(diffuse=(0.7, 0.6, 0.5), specular=(0.2, 0.2, 0.2), shininess=32.0, alpha=1.0)
    lo, hi, n = 0.1, 0.9, 9
    g = [lo + (hi - lo) * i / n for i in range(n + 1)]
    tris = []
    # (fixed axis, fixed value, u axis, v axis) with u x v pointing outward
    faces = [(0, hi, 1, 2), (0, lo, 2, 1), (1, hi, 2, 0), (1, lo, 0, 2), (2, hi, 0, 1), (2, lo, 1, 0)]
    for obj, (ax, val, ua, va) in enumerate(faces):
        for i in range(n):
            for j in range(n):
                def P(a, b):
                    p = [0.0, 0.0, 0.0]
                    p[ax] = val
                    p[ua] = g[a]
                    p[va] = g[b]
                    return tuple(p)
                tris += make_quad(P(i, j), P(i + 1, j), P(i + 1, j + 1), P(i, j + 1), 0, obj)
    return Scene.from_triangles(tris, [mat])


def sphere_field(n_spheres: int, subdivisions: int, seed: int, r_lo: float, r_hi: float,
                 c_lo: float, c_hi: float, alpha: float = 1.0) -> Scene:
    """Random field of icospheres, built struct-of-arrays.

    Per sphere ``k``: centre ~ U[c_lo, c_hi]^3, radius ~ U[r_lo, r_hi] from
    ``np.random.default_rng(seed)``; object id k and material k.  Values are
    bit-identical to ``make_triangle(c + r*v[a], c + r*v[b], c + r*v[c],
    v[a], v[b], v[c])`` per face (same operation sequence, vectorised).
    """
    rng = np.random.default_rng(seed)
    centers = rng.uniform(c_lo, c_hi, size=(n_spheres, 3))
    radii = rng.uniform(r_lo, r_hi, size=n_spheres)
    colors = rng.uniform(0.2, 0.9, size=(n_spheres, 3))
    verts, faces = icosphere_mesh(subdivisions)
    V = np.array(verts)                                   # (nv, 3)
    F = np.array(faces, dtype=np.int64)                   # (nf, 3)
    # make_triangle re-normalises the given vertex normals: unit(v) = v / sqrt(v @ v)
    Vn = V / np.sqrt(np.vecdot(V, V))[:, None]
    nf = len(F)
    T = n_spheres * nf
    pos = np.empty((T, 3, 3))
    for k in range(n_spheres):
        pos[k * nf:(k + 1) * nf] = centers[k] + radii[k] * V[F]
    nrm = np.broadcast_to(Vn[F][None], (n_spheres, nf, 3, 3)).reshape(T, 3, 3)
    cr = np.cross(pos[:, 1] - pos[:, 0], pos[:, 2] - pos[:, 0])
    length = np.sqrt(np.vecdot(cr, cr))
    fn = np.zeros_like(cr)
    ok = length > 0.0
    fn[ok] = cr[ok] / length[ok, None]
    mats = [Material(diffuse=tuple(float(c) for c in colors[k]), specular=(0.25, 0.25, 0.25),
                     shininess=24.0, alpha=alpha) for k in range(n_spheres)]
    ids = np.repeat(np.arange(n_spheres, dtype=np.uint32), nf)
    return Scene.from_arrays(pos, nrm, fn, ids, ids, mats)


def spheres100k() -> Scene:
    """C2: 5 icospheres (subdivision 5) = 102,400 triangles, seed 0."""
    return sphere_field(5, 5, seed=0, r_lo=0.05, r_hi=0.2, c_lo=0.2, c_hi=0.8, alpha=0.6)


def scatter1m() -> Scene:
    """C3: 48 icospheres (subdivision 5) = 983,040 triangles, seed 1."""
    return sphere_field(48, 5, seed=1, r_lo=0.02, r_hi=0.12, c_lo=0.15, c_hi=0.85, alpha=1.0)


def layers80(n: int = 80) -> Scene:
    """C4: depth-complex stack of n translucent quads (alpha 0.05) at
    z_k = 0.1 + 0.8 k/(n-1), inset 0.02 (k mod 5); material = object = k."""
    mats, tris = [], []
    for k in range(n):
        z = 0.1 + 0.8 * k / (n - 1)
        a, b = 0.05 + 0.02 * (k % 5), 0.95 - 0.02 * (k % 5)
        mats.append(Material(diffuse=(0.2 + 0.6 * (k % 3) / 2, 0.5, 0.8 - 0.6 * (k % 4) / 3), alpha=0.05))
        tris += make_quad((a, a, z), (b, a, z), (b, b, z), (a, b, z), material_id=k, object_id=k)
    return Scene.from_triangles(tris, mats)


def c5_views(n: int = 64, resolution=(3840, 2160), distance: float = 1.5, fov_deg: float = 45.0, seed: int = 2):
    """BASELINE config C5's novel viewpoints: n cameras on
    a Fibonacci sphere (random rotation from default_rng(seed)) at `distance`
    from the cube centre, looking at it, fov 45, 4K."""
    from .scene import look_at_camera
    rng = np.random.default_rng(seed)
    phi0 = rng.uniform(0.0, 2.0 * np.pi)
    golden = np.pi * (3.0 - np.sqrt(5.0))
    views = []
    for i in range(n):
        z = 1.0 - 2.0 * (i + 0.5) / n
        r = np.sqrt(max(0.0, 1.0 - z * z))
        a = phi0 + golden * i
        d = np.array([r * np.cos(a), r * np.sin(a), z])
        up = (0.0, 0.0, 1.0) if abs(z) < 0.9 else (0.0, 1.0, 0.0)
        views.append(look_at_camera(0.5 + distance * d, up=up, resolution=resolution, fov_deg=fov_deg))
    return views
