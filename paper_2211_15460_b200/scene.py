"""Scenes, materials and cameras -- host-side inputs of the capture path.

Mirrors the reference's scene model (``fhv/scene.py``) so that a user of the
reference can hand the same triangles to this package.  The difference is the
storage: a :class:`Scene` here is struct-of-arrays (``positions[T,3,3]``,
``normals[T,3,3]``, ``face_normals[T,3]``, ``material_id[T]``,
``object_id[T]``), which is the layout uploaded to HBM; per-triangle
:class:`Triangle` objects are materialised only on demand.

Bit-exactness of the inputs matters because coverage ties are decided in
exact f64: :func:`make_triangle` performs the same IEEE operations as the
reference (``fhv/scene.py:129-145``), so face normals are bit-identical.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "AXIS_VIEWS", "Aabb", "Camera", "Material", "Scene", "SceneError", "SceneLoadError",
    "SceneTransform", "Triangle", "Vertex", "capture_camera", "make_quad", "make_triangle", "normalize_scene",
    "viewpoint_camera", "DEFAULT_MATERIAL_NAME", "load_material_table", "load_scene", "save_material_table",
    "save_scene",
]

# Capture frames look down the negative axis with a pinned up vector
# (fhv/scene.py:46-52).
AXIS_VIEWS = {
    "+x": ((-1.0, 0.0, 0.0), (0.0, 1.0, 0.0)),
    "+y": ((0.0, -1.0, 0.0), (0.0, 0.0, 1.0)),
    "+z": ((0.0, 0.0, -1.0), (0.0, 1.0, 0.0)),
}


class SceneError(ValueError):
    """Invalid scene content or geometry (fhv/scene.py:55-56)."""


class SceneLoadError(SceneError):
    def __init__(self, path, line_no: int, message: str):
        super().__init__(f"{path}:{line_no}: {message}")
        self.path = str(path)
        self.line_no = line_no


def _as3(v) -> np.ndarray:
    a = np.asarray(v, dtype=np.float64)
    if a.shape != (3,):
        raise SceneError(f"expected 3-vector, got shape {a.shape}")
    return a


def _normalized(v: np.ndarray) -> np.ndarray:
    # sqrt(v @ v): a BLAS ddot, i.e. the FWD fma chain
    length = math.sqrt(float(v @ v))
    if length == 0.0:
        raise SceneError("zero-length direction")
    return v / length


@dataclass(frozen=True)
class Material:
    """Blinn-Phong material with straight alpha (fhv/scene.py:82-96)."""

    diffuse: tuple = (0.8, 0.8, 0.8)
    specular: tuple = (0.0, 0.0, 0.0)
    shininess: float = 32.0
    alpha: float = 1.0

    def __post_init__(self):
        for channel in (*self.diffuse, *self.specular):
            if not 0.0 <= channel <= 1.0:
                raise SceneError(f"material channel {channel} outside [0,1]")
        if not self.shininess > 0.0:
            raise SceneError("shininess must be > 0")
        if not 0.0 <= self.alpha <= 1.0:
            raise SceneError(f"alpha {self.alpha} outside [0,1]")


@dataclass
class Vertex:
    position: np.ndarray
    normal: np.ndarray


@dataclass
class Triangle:
    v0: Vertex
    v1: Vertex
    v2: Vertex
    material_id: int = 0
    object_id: int = 0
    face_normal: np.ndarray = field(default_factory=lambda: np.zeros(3))

    @property
    def positions(self) -> np.ndarray:
        return np.stack([self.v0.position, self.v1.position, self.v2.position])

    @property
    def normals(self) -> np.ndarray:
        return np.stack([self.v0.normal, self.v1.normal, self.v2.normal])

    @property
    def area(self) -> float:
        e = np.cross(self.v1.position - self.v0.position, self.v2.position - self.v0.position)
        return 0.5 * float(np.linalg.norm(e))


def make_triangle(p0, p1, p2, n0=None, n1=None, n2=None, material_id: int = 0,
                  object_id: int = 0) -> Triangle:
    """Triangle with the face normal as default vertex normal.

    Same IEEE operations as fhv/scene.py:129-145: np.cross of the two edges,
    divided by its ddot norm; zero-area faces keep a zero face normal.
    """
    a, b, c = _as3(p0), _as3(p1), _as3(p2)
    cr = np.cross(b - a, c - a)
    length = float(np.linalg.norm(cr))
    fn = cr / length if length > 0.0 else np.zeros(3)
    verts = [Vertex(p, fn if n is None else _normalized(_as3(n))) for p, n in ((a, n0), (b, n1), (c, n2))]
    return Triangle(*verts, material_id=material_id, object_id=object_id, face_normal=fn)


def make_quad(p00, p10, p11, p01, material_id: int = 0, object_id: int = 0) -> list:
    """Two triangles sharing the (p00, p11) diagonal (fhv/scene.py:148-153)."""
    return [make_triangle(p00, p10, p11, material_id=material_id, object_id=object_id),
            make_triangle(p00, p11, p01, material_id=material_id, object_id=object_id)]


@dataclass(frozen=True)
class Aabb:
    lo: np.ndarray
    hi: np.ndarray

    @staticmethod
    def from_points(points) -> "Aabb":
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
        return Aabb(pts.min(axis=0), pts.max(axis=0))

    @property
    def center(self) -> np.ndarray:
        return 0.5 * (self.lo + self.hi)

    @property
    def extent(self) -> np.ndarray:
        return self.hi - self.lo

    def contains(self, points) -> bool:
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
        return bool(np.all(pts >= self.lo) and np.all(pts <= self.hi))


class Scene:
    """Triangle soup + material table, stored struct-of-arrays.

    ``Scene(triangles, materials, bounds)`` keeps the reference's dataclass
    signature (fhv/scene.py:179-198); :meth:`from_arrays` is the bulk path.
    """

    def __init__(self, triangles=None, materials=None, bounds: Aabb | None = None, *,
                 arrays: dict | None = None):
        if arrays is None:
            tris = list(triangles or [])
            T = len(tris)
            arrays = {
                "positions": np.array([t.positions for t in tris], dtype=np.float64).reshape(T, 3, 3),
                "normals": np.array([t.normals for t in tris], dtype=np.float64).reshape(T, 3, 3),
                "face_normals": np.array([t.face_normal for t in tris], dtype=np.float64).reshape(T, 3),
                "material_id": np.array([t.material_id for t in tris], dtype=np.uint32),
                "object_id": np.array([t.object_id for t in tris], dtype=np.uint32),
            }
            self._triangles = tris
        else:
            self._triangles = None
        self.positions = np.ascontiguousarray(arrays["positions"], dtype=np.float64)
        self.normals = np.ascontiguousarray(arrays["normals"], dtype=np.float64)
        self.face_normals = np.ascontiguousarray(arrays["face_normals"], dtype=np.float64)
        self.material_id = np.ascontiguousarray(arrays["material_id"], dtype=np.uint32)
        self.object_id = np.ascontiguousarray(arrays["object_id"], dtype=np.uint32)
        self.materials = list(materials) if materials else [Material()]
        if bounds is None:
            bounds = Aabb.from_points(self.positions) if len(self.positions) else Aabb(np.zeros(3), np.zeros(3))
        self.bounds = bounds

    @staticmethod
    def from_triangles(triangles, materials=None) -> "Scene":
        tris = list(triangles)
        if not tris:
            raise SceneError("scene has no triangles")
        mats = list(materials) if materials else [Material()]
        for t in tris:
            if t.material_id >= len(mats):
                raise SceneError(f"material_id {t.material_id} out of range")
        return Scene(tris, mats)

    @staticmethod
    def from_arrays(positions, normals, face_normals, material_id, object_id, materials=None) -> "Scene":
        T = len(positions)
        if T == 0:
            raise SceneError("scene has no triangles")
        mats = list(materials) if materials else [Material()]
        mid = np.asarray(material_id, dtype=np.uint32).reshape(T)
        if int(mid.max()) >= len(mats):
            raise SceneError("material_id out of range")
        return Scene(materials=mats, arrays={
            "positions": np.asarray(positions).reshape(T, 3, 3),
            "normals": np.asarray(normals).reshape(T, 3, 3),
            "face_normals": np.asarray(face_normals).reshape(T, 3),
            "material_id": mid,
            "object_id": np.asarray(object_id, dtype=np.uint32).reshape(T),
        })

    @property
    def n_triangles(self) -> int:
        return int(self.positions.shape[0])

    @property
    def triangles(self) -> list:
        if self._triangles is None:
            self._triangles = [
                Triangle(Vertex(p[0].copy(), n[0].copy()), Vertex(p[1].copy(), n[1].copy()),
                         Vertex(p[2].copy(), n[2].copy()), int(m), int(o), f.copy())
                for p, n, f, m, o in zip(self.positions, self.normals, self.face_normals,
                                         self.material_id, self.object_id)]
        return self._triangles

    @property
    def n_objects(self) -> int:
        n = self.__dict__.get("_n_objects")
        if n is None:
            n = self.__dict__["_n_objects"] = int(len(np.unique(self.object_id)))
        return n


class Camera:
    """Orthographic or perspective camera (fhv/scene.py:201-244).

    ``extent_or_fov`` is the view-volume height (orthographic) or the
    vertical field of view in degrees (perspective).  Raster origin is the
    top-left corner; ``up`` maps to decreasing raster y.
    """

    def __init__(self, kind, eye, view_dir, up, extent_or_fov, resolution, near, far):
        if kind not in ("orthographic", "perspective"):
            raise SceneError(f"unknown camera kind {kind!r}")
        self.kind = kind
        self.eye = _as3(eye)
        self.view_dir = _normalized(_as3(view_dir))
        self.up = _normalized(_as3(up))
        self.extent_or_fov = float(extent_or_fov)
        self.resolution = (int(resolution[0]), int(resolution[1]))
        self.near = float(near)
        self.far = float(far)
        if self.resolution[0] < 1 or self.resolution[1] < 1:
            raise SceneError("resolution must be >= 1")
        if not self.near < self.far:
            raise SceneError("near must be < far")
        if self.extent_or_fov <= 0.0:
            raise SceneError("extent/fov must be > 0")

    def basis(self):
        """(right, up, forward), up re-orthogonalised."""
        f = self.view_dir
        r = _normalized(np.cross(f, self.up))
        return r, np.cross(r, f), f

    @property
    def aspect(self) -> float:
        return self.resolution[0] / self.resolution[1]

    def scalars(self) -> np.ndarray:
        """Camera packed for the device kernels (and the oracle):
        [persp, eye3, r3, u3, f3, w, h, half_w, half_h, tan(fov/2), aspect,
        near, far, extent].  Every derived scalar is computed with the same
        Python expression the reference uses (fhv/render.py:211-242,
        fhv/raycast.py:148-172).  Cached per camera state (read-only array)."""
        key = (self.kind, self.eye.tobytes(), self.view_dir.tobytes(), self.up.tobytes(), self.extent_or_fov,
               self.resolution, self.near, self.far)
        hit = self.__dict__.get("_scalars")
        if hit is not None and hit[0] == key:
            return hit[1]
        r, u, f = self.basis()
        w, h = self.resolution
        persp = self.kind == "perspective"
        half_h = self.extent_or_fov / 2.0
        half_w = half_h * self.aspect
        t = math.tan(math.radians(self.extent_or_fov) / 2.0) if persp else 0.0
        out = np.array([1.0 if persp else 0.0, *self.eye, *r, *u, *f, w, h, half_w, half_h, t,
                        self.aspect, self.near, self.far, self.extent_or_fov], dtype=np.float64)
        out.flags.writeable = False
        self.__dict__["_scalars"] = (key, out)
        return out


@dataclass(frozen=True)
class SceneTransform:
    """Uniform scale followed by translation: p' = scale * p + offset (fhv/scene.py:441-457)."""

    scale: float
    offset: np.ndarray

    def apply(self, points) -> np.ndarray:
        return np.asarray(points, dtype=np.float64) * self.scale + self.offset

    def invert(self, points) -> np.ndarray:
        return (np.asarray(points, dtype=np.float64) - self.offset) / self.scale

    @property
    def is_identity(self) -> bool:
        return self.scale == 1.0 and not self.offset.any()


def normalize_scene(scene: Scene, margin: float = 0.0):
    """Uniformly map the scene bounds into [margin, 1-margin]^3 (fhv/scene.py:460-487),
    vectorised over all vertices (same elementwise p * scale + offset).
    Returns the normalised scene and its SceneTransform."""
    if not 0.0 <= margin < 0.25:
        raise SceneError(f"margin {margin} outside [0, 0.25)")
    longest = float(scene.bounds.extent.max())
    if longest == 0.0:
        raise SceneError("degenerate scene bounds (zero extent on all axes)")
    scale = (1.0 - 2.0 * margin) / longest
    offset = 0.5 - scale * scene.bounds.center
    pos = scene.positions * scale + offset
    out = Scene(materials=scene.materials, arrays={
        "positions": pos, "normals": scene.normals, "face_normals": scene.face_normals,
        "material_id": scene.material_id, "object_id": scene.object_id})
    return out, SceneTransform(scale, offset)


def capture_camera(scene: Scene, axis: str = "+z", resolution: int = 256) -> Camera:
    """Orthographic capture camera over the unit cube (fhv/scene.py:490-508)."""
    if axis not in AXIS_VIEWS:
        raise SceneError(f"unknown capture axis {axis!r}")
    view_dir, up = AXIS_VIEWS[axis]
    return Camera("orthographic", scene.bounds.center, np.array(view_dir), np.array(up), 1.0,
                  (resolution, resolution), -1.0, 1.0)


def viewpoint_camera(axis: str = "+z", resolution=(256, 256), kind: str = "orthographic",
                     fov_deg: float = 45.0, distance: float = 1.5, center=(0.5, 0.5, 0.5)) -> Camera:
    """Camera outside the unit cube looking back at its centre (fhv/scene.py:511-524)."""
    if axis not in AXIS_VIEWS:
        raise SceneError(f"unknown axis {axis!r}")
    view_dir, up = AXIS_VIEWS[axis]
    eye = _as3(center) + distance * -np.array(view_dir)
    if kind == "orthographic":
        return Camera(kind, eye, np.array(view_dir), np.array(up), 1.0, resolution, 0.0, distance + 1.0)
    return Camera(kind, eye, np.array(view_dir), np.array(up), fov_deg, resolution, 1e-3, distance + 1.0)


def look_at_camera(eye, target=(0.5, 0.5, 0.5), up=(0.0, 1.0, 0.0), resolution=(1920, 1080),
                   fov_deg: float = 45.0, near: float = 1e-3, far: float = 3.0) -> Camera:
    """Perspective camera at ``eye`` looking at ``target`` (bench view batches)."""
    eye = _as3(eye)
    d = _as3(target) - eye
    return Camera("perspective", eye, d, _as3(up), fov_deg, resolution, near, far)


# scene files at the reference's module path (fhv/scene.py:251-432); the
# implementation is ingest.py (bulk parse, device normalisation)
DEFAULT_MATERIAL_NAME = "__default__"


def load_material_table(path):
    from .ingest import load_material_table as f
    return f(path)


def load_scene(path, material_table=None, device=None):
    from .ingest import load_scene as f
    return f(path, material_table, device)


def save_material_table(materials, names, path) -> None:
    from .ingest import save_material_table as f
    return f(materials, names, path)


def save_scene(scene, path, material_path=None) -> None:
    from .ingest import save_scene as f
    return f(scene, path, material_path)
