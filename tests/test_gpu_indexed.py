"""The indexed-mesh upload bench.py's e2e line uses (device.IndexedMesh ->
IndexedUpload -> DeviceScene.load_indexed, kernel k_expand_indexed): the
triangle arrays it rebuilds on the device must be byte-identical to the
directly uploaded ones (DeviceScene(scene)), face normals included, and a bad
vertex index must be refused before anything is uploaded (the kernel's own
bounds check only guards the device)."""
import numpy as np
import pytest
import torch

from paper_2211_15460_b200 import sample_scenes
from paper_2211_15460_b200.device import DeviceScene, IndexedMesh, IndexedUpload

DEV = torch.device("cuda", 0)


def _bits(t):
    return t.view(torch.int64) if t.dtype == torch.float64 else t


def _load(scene):
    mesh = IndexedMesh.from_scene(scene)
    up = IndexedUpload(mesh, DEV)
    for d, src in zip(up.tensors(), mesh.arrays()):
        d.copy_(torch.from_numpy(np.ascontiguousarray(src)))
    ds = DeviceScene(scene, DEV)
    for f in ("pos", "vnrm", "fnrm", "mat", "obj"):
        getattr(ds, f).zero_()
    return mesh, up, ds


@pytest.mark.gpu
@pytest.mark.parametrize("name", ("small", "scatter1m"))
def test_indexed_expansion_byte_identical(name):
    scene = (sample_scenes.sphere_field(5, 2, seed=11, r_lo=0.05, r_hi=0.2, c_lo=0.2, c_hi=0.8) if name == "small"
             else sample_scenes.scatter1m())
    mesh, up, ds = _load(scene)
    assert mesh.n_vertices < 3 * scene.n_triangles  # shared corners were merged
    ds.load_indexed(up)
    ref = DeviceScene(scene, DEV)
    torch.cuda.synchronize()
    for f in ("pos", "vnrm", "fnrm", "mat", "obj"):
        assert torch.equal(_bits(getattr(ds, f)), _bits(getattr(ref, f))), f


def test_indexed_bad_vertex_index_rejected():
    scene = sample_scenes.sphere_field(3, 1, seed=2, r_lo=0.05, r_hi=0.2, c_lo=0.2, c_hi=0.8)
    m = IndexedMesh.from_scene(scene)
    faces = m.faces.copy()
    faces[1, 2] = m.n_vertices  # one past the end
    with pytest.raises(ValueError):
        IndexedMesh(m.vpos, m.vn, faces, m.mat, m.obj)
