"""Scene ingest at 1 M-triangle scale:
``load_scene`` / ``load_material_table`` / ``save_scene`` /
``save_material_table`` of the reference (fhv/scene.py:251-432), same file
format, same errors (``SceneLoadError`` with file:line), bit-identical Scene
arrays.

The reference parses line by line and calls ``make_triangle`` per face
(NumPy per triangle, tens of microseconds each).  Here one pass over the
lines only tokenises and validates (the checks the reference makes, in file
order, so the first error reported is the same); the geometry is then built
in bulk: fan triangulation with NumPy index arithmetic, and the f64
normalisations on the device with the reference's operation order
(``np.linalg.norm`` / ``_unit`` = sqrt of a ddot, then an IEEE divide:
``fhv_unit_rows``; face normals = ``make_triangle``'s cross / norm:
``fhv_face_normals``) -- no CPU fallback.
"""
from __future__ import annotations

import ctypes
import math
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .device import default_device
from .scene import DEFAULT_MATERIAL_NAME, Material, Scene, SceneError, SceneLoadError

__all__ = ["DEFAULT_MATERIAL_NAME", "load_material_table", "load_scene", "save_material_table", "save_scene"]


def load_material_table(path) -> tuple[list, dict]:
    """Parse a material table (fhv/scene.py:251-278).  Returns (materials, name -> index)."""
    materials: list = []
    names: dict = {}
    with open(path, "r", encoding="utf-8") as fh:
        for line_no, raw in enumerate(fh, start=1):
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            if len(parts) != 9:
                raise SceneLoadError(path, line_no, f"expected 9 fields, got {len(parts)}")
            name = parts[0]
            try:
                vals = [float(p) for p in parts[1:]]
            except ValueError as exc:
                raise SceneLoadError(path, line_no, str(exc)) from None
            if not all(math.isfinite(v) for v in vals):
                raise SceneLoadError(path, line_no, "non-finite value")
            if name in names:
                raise SceneLoadError(path, line_no, f"duplicate material {name!r}")
            try:
                mat = Material(tuple(vals[0:3]), tuple(vals[3:6]), vals[6], vals[7])
            except SceneError as exc:
                raise SceneLoadError(path, line_no, str(exc)) from None
            names[name] = len(materials)
            materials.append(mat)
    return materials, names


def _floats(parts, path, line_no):
    try:
        vals = [float(p) for p in parts]
    except ValueError as exc:
        raise SceneLoadError(path, line_no, str(exc)) from None
    if not all(math.isfinite(v) for v in vals):
        raise SceneLoadError(path, line_no, "non-finite coordinate")
    return vals


def _unit_rows(a: np.ndarray, dev) -> tuple[np.ndarray, int]:
    """Device rows / sqrt(row . row) (FWD ddot order); (result, first zero row or -1)."""
    if len(a) == 0:
        return np.zeros((0, 3)), -1
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
    out = torch.empty_like(t)
    z = ctypes.c_int64(-1)
    rc = _lib.load().fhv_unit_rows(_lib.ctx(dev), len(a), _lib.ptr(t), _lib.ptr(out), ctypes.byref(z),
                                   _lib.stream_ptr(dev))
    _lib.check(rc, "unit rows")
    return out.cpu().numpy(), int(z.value)


def load_scene(path, material_table=None, device=None) -> Scene:
    """Load a scene file (fhv/scene.py:291-378), fan-triangulating faces.

    Faces carry the object id of their enclosing named group (numbered in
    order of first use by a face) and the material selected by the last
    ``usemtl``; both default to 0 / a default material appended on first
    use.  Vertex normals given by ``vn`` are unit-normalised at load and
    again by ``make_triangle``; corners without one take the face normal.
    """
    if material_table is not None:
        materials, mat_names = load_material_table(material_table)
    else:
        materials, mat_names = [], {}
    v_vals: list = []       # flat x, y, z per position
    vn_vals: list = []      # flat raw normal components
    corner_v: list = []     # 0-based position index per face corner
    corner_n: list = []     # 0-based normal index per corner, or -1
    face_len: list = []     # corners per face
    face_mat: list = []
    face_obj: list = []
    object_ids: dict = {}
    current_group = ""
    current_material = None
    default_material = None
    n_pos = n_nrm = 0
    pending = None  # the first SceneLoadError: faces before its line still build (and may raise first)
    with open(path, "r", encoding="utf-8") as fh:
        try:
            for line_no, raw in enumerate(fh, start=1):
                line = raw.strip()
                if not line or line[0] == "#":
                    continue
                key, *parts = line.split()
                if key == "f":
                    if len(parts) < 3:
                        raise SceneLoadError(path, line_no, "face needs >= 3 vertices")
                    for token in parts:
                        fields = token.split("/")
                        nf = len(fields)
                        if (nf != 1 and nf != 3) or (nf == 3 and fields[1]):
                            raise SceneLoadError(path, line_no, f"bad face token {token!r}")
                        try:
                            vi = int(fields[0])
                            ni = int(fields[2]) if nf == 3 and fields[2] else None
                        except ValueError:
                            raise SceneLoadError(path, line_no, f"bad face token {token!r}") from None
                        if not 1 <= vi <= n_pos:
                            raise SceneLoadError(path, line_no, f"vertex index {vi} out of range")
                        if ni is not None and not 1 <= ni <= n_nrm:
                            raise SceneLoadError(path, line_no, f"normal index {ni} out of range")
                        corner_v.append(vi - 1)
                        corner_n.append(-1 if ni is None else ni - 1)
                    face_len.append(len(parts))
                    if current_material is not None:
                        mat_id = current_material
                    else:
                        if default_material is None:
                            default_material = len(materials)
                            materials.append(Material())
                            mat_names[DEFAULT_MATERIAL_NAME] = default_material
                        mat_id = default_material
                    face_mat.append(mat_id)
                    obj = object_ids.get(current_group)
                    if obj is None:
                        obj = object_ids[current_group] = len(object_ids)
                    face_obj.append(obj)
                elif key == "v":
                    if len(parts) != 3:
                        raise SceneLoadError(path, line_no, "v needs 3 coordinates")
                    v_vals += _floats(parts, path, line_no)
                    n_pos += 1
                elif key == "vn":
                    if len(parts) != 3:
                        raise SceneLoadError(path, line_no, "vn needs 3 coordinates")
                    x, y, z = _floats(parts, path, line_no)
                    # np.linalg.norm == 0 exactly when every square rounds to 0 (the
                    # ddot's terms are non-negative): checked here, in file order
                    if x * x == 0.0 and y * y == 0.0 and z * z == 0.0:
                        raise SceneLoadError(path, line_no, "zero-length normal")
                    vn_vals += (x, y, z)
                    n_nrm += 1
                elif key == "g":
                    current_group = parts[0] if parts else ""
                elif key == "usemtl":
                    if len(parts) != 1:
                        raise SceneLoadError(path, line_no, "usemtl needs a name")
                    if parts[0] not in mat_names:
                        raise SceneLoadError(path, line_no, f"unknown material {parts[0]!r}")
                    current_material = mat_names[parts[0]]
                else:
                    raise SceneLoadError(path, line_no, f"unknown keyword {key!r}")
        except SceneLoadError as err:
            pending = err
    vn_raw = np.asarray(vn_vals, dtype=np.float64).reshape(-1, 3)
    # a vn whose squared norm overflows normalises to 0 at load (n / inf);
    # make_triangle's _unit then raises SceneError at the first face (file
    # order) using it (fhv/scene.py:75-78) -- before any later line is parsed,
    # so before a pending SceneLoadError of a later line
    if len(vn_raw):
        cn_all = np.asarray(corner_n[:sum(face_len)], dtype=np.int64)  # corners of completed faces
        with np.errstate(over="ignore"):
            zero_row = np.isinf(np.einsum("ij,ij->i", vn_raw, vn_raw))
        bad = (cn_all >= 0) & zero_row[np.maximum(cn_all, 0)]
        if bad.any():
            raise SceneError("zero-length direction")
    if pending is not None:
        raise pending
    if not face_len:
        raise SceneLoadError(path, 0, "empty scene (no faces)")
    if not materials:
        materials.append(Material())
    dev = default_device(device)
    P = np.asarray(v_vals, dtype=np.float64).reshape(-1, 3)
    # vn normalisation at load (n / np.linalg.norm(n)); zero rows were rejected above
    vn, zero = _unit_rows(vn_raw, dev)
    assert zero < 0
    # make_triangle's _unit of each given normal (per distinct normal: deterministic)
    vn_u, _ = _unit_rows(vn, dev)
    # fan triangulation: face corners c0..ck -> (c0, ci, ci+1)
    flen = np.asarray(face_len, dtype=np.int64)
    start = np.concatenate(([0], np.cumsum(flen)[:-1]))
    ntri = flen - 2
    tri_face = np.repeat(np.arange(len(flen)), ntri)
    k = np.arange(int(ntri.sum())) - np.repeat(np.cumsum(ntri) - ntri, ntri)  # 0..ntri-1 within each face
    c0 = start[tri_face]
    c1 = c0 + 1 + k
    corners = np.stack([c0, c1, c1 + 1], axis=1)
    cv = np.asarray(corner_v, dtype=np.int64)[corners]
    cn = np.asarray(corner_n, dtype=np.int64)[corners]
    pos = np.ascontiguousarray(P[cv])  # (T, 3, 3)
    # face normals exactly as make_triangle (cross, sqrt(ddot), divide; 0 when degenerate)
    tp = torch.from_numpy(pos).to(dev)
    fn = torch.empty((len(pos), 3), dtype=torch.float64, device=dev)
    rc = _lib.load().fhv_face_normals(_lib.ctx(dev), len(pos), _lib.ptr(tp), _lib.ptr(fn), _lib.stream_ptr(dev))
    _lib.check(rc, "face normals")
    fnrm = fn.cpu().numpy()
    nrm = np.where((cn >= 0)[..., None], vn_u[np.maximum(cn, 0)] if len(vn_u) else 0.0, fnrm[:, None, :])
    mat = np.asarray(face_mat, dtype=np.uint32)[tri_face]
    obj = np.asarray(face_obj, dtype=np.uint32)[tri_face]
    return Scene.from_arrays(pos, np.ascontiguousarray(nrm), fnrm, mat, obj, materials)


def save_material_table(materials, names, path) -> None:
    """fhv/scene.py:381-388."""
    lines = []
    for name, m in zip(names, materials):
        lines.append(" ".join([name] + [f"{v:.9g}" for v in (*m.diffuse, *m.specular, m.shininess, m.alpha)]))
    Path(path).write_text("\n".join(lines) + "\n", encoding="utf-8")


def save_scene(scene: Scene, path, material_path=None) -> None:
    """Write a scene in the loader's format (fhv/scene.py:391-432): exact
    vertex / normal dedup in first-use order, ``g obj<id>`` + ``usemtl m<id>``
    whenever (object, material) changes, ``f p//n`` faces."""
    T = scene.n_triangles
    P = np.ascontiguousarray(scene.positions.reshape(T * 3, 3))
    N = np.ascontiguousarray(scene.normals.reshape(T * 3, 3))

    def dedup(a):
        # first-use order of exact (bitwise) rows, like dict insertion order on tuple(p.tolist())
        # (-0.0 and 0.0 compare equal as Python floats: canonicalise before hashing)
        canon = a + 0.0
        _, first, inv = np.unique(canon.view(np.dtype((np.void, 24))), return_index=True, return_inverse=True)
        order = np.argsort(first, kind="stable")
        rank = np.empty_like(order)
        rank[order] = np.arange(len(order))
        return a[np.sort(first)], rank[inv.reshape(-1)] + 1

    pu, pid = dedup(P)
    nu, nid = dedup(N)
    lines = ["v " + " ".join(f"{c:.17g}" for c in row) for row in pu.tolist()]
    lines += ["vn " + " ".join(f"{c:.17g}" for c in row) for row in nu.tolist()]
    obj, mat = scene.object_id, scene.material_id
    pid, nid = pid.reshape(T, 3), nid.reshape(T, 3)
    current = None
    for t in range(T):
        key = (int(obj[t]), int(mat[t]))
        if key != current:
            lines.append(f"g obj{key[0]}")
            lines.append(f"usemtl m{key[1]}")
            current = key
        lines.append("f " + " ".join(f"{pid[t, i]}//{nid[t, i]}" for i in range(3)))
    Path(path).write_text("\n".join(lines) + "\n", encoding="utf-8")
    if material_path is not None:
        save_material_table(scene.materials, [f"m{i}" for i in range(len(scene.materials))], material_path)
