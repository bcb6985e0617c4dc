"""Helpers to read the committed golden vectors (tests/golden/*.npz)."""
import functools
import hashlib
import json
import os

import numpy as np

from paper_2211_15460_b200.scene import Material, Scene

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def npz(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


@functools.lru_cache(maxsize=None)
def meta():
    return json.load(open(os.path.join(GOLDEN, "golden_meta.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def golden_scene(name):
    """Scene rebuilt from the reference's own triangle arrays (host-BLAS independent)."""
    g = npz("scenes")
    k = name + "/"
    mats = [Material(tuple(d), tuple(s), float(h), float(a)) for d, s, h, a in
            zip(g[k + "mat_diffuse"], g[k + "mat_specular"], g[k + "mat_shininess"], g[k + "mat_alpha"])]
    return Scene.from_arrays(g[k + "positions"], g[k + "normals"], g[k + "face_normals"],
                             g[k + "material_id"], g[k + "object_id"], mats)


BUILTINS = ("cornell", "edge-plane", "icosphere", "three-quads")
