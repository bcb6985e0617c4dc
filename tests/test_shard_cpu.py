"""Host logic of the multi-GPU partition (paper_2211_15460_b200/shard.py) on
CPU: Morton ranges and their world-space covers, and the exchange layer over
torch.distributed (gloo, world_size 2) and the in-process loopback."""
import os
import socket
import threading

import numpy as np
import pytest
import torch

from paper_2211_15460_b200 import sample_scenes, shard
from paper_2211_15460_b200.raster import CaptureStrategy, RasterConfig
from paper_2211_15460_b200.scene import capture_camera
from paper_2211_15460_b200.storage import FhvError, morton_decode


@pytest.mark.parametrize("levels", (4, 5, 6, 8))
@pytest.mark.parametrize("world", (1, 2, 3, 4, 8))
def test_ranges_tile_the_directory(levels, world):
    tl = shard.tile_leaves(levels)
    if world > 8 ** levels // tl:
        with pytest.raises(FhvError):
            shard.shard_ranges(levels, world)
        return
    r = shard.shard_ranges(levels, world)
    assert r[0][0] == 0 and r[-1][1] == 8 ** levels
    for (a, b), (c, _) in zip(r, r[1:]):
        assert b == c
    for a, b in r:
        assert a % tl == 0 and b % tl == 0 and b > a


def test_balanced_ranges_follow_weights():
    levels = 8
    n_tiles = 8 ** levels // shard.tile_leaves(levels)
    w = np.zeros(n_tiles)
    w[:10] = 100.0  # all the work in the first tiles
    r = shard.shard_ranges(levels, 4, w)
    assert r[0][0] == 0 and r[-1][1] == 8 ** levels
    assert all(b > a for a, b in r)
    tl = shard.tile_leaves(levels)
    sizes = [(b - a) // tl for a, b in r]
    assert sizes[0] < 10 and sum(sizes[:3]) <= 10  # the heavy tiles are split across ranks
    with pytest.raises(FhvError):
        shard.shard_ranges(levels, 2, np.ones(3))


@pytest.mark.parametrize("levels", (4, 6))
def test_range_boxes_cover_exactly_the_range(levels):
    rng = np.random.default_rng(0)
    tl = shard.tile_leaves(levels)
    n_tiles = 8 ** levels // tl
    for _ in range(20):
        a, b = sorted(rng.choice(n_tiles + 1, 2, replace=False))
        lo, hi = int(a) * tl, int(b) * tl
        boxes = shard.range_boxes(lo, hi, levels)
        assert 1 <= len(boxes) <= shard.MAX_BOXES
        # every leaf centre inside the range is covered, every covered leaf is in the range
        codes = np.arange(8 ** levels)
        x, y, z = morton_decode(codes, levels)
        c = (np.stack([x, y, z], 1) + 0.5) / (1 << levels)
        inside = np.zeros(len(codes), bool)
        for bx in boxes:
            inside |= np.all((c >= bx[:3]) & (c <= bx[3:]), axis=1)
        want = (codes >= lo) & (codes < hi)
        if len(boxes) < shard.MAX_BOXES:
            assert np.array_equal(inside, want)
        else:
            assert np.all(inside[want])


def test_fragment_weights_shape_and_total():
    s = sample_scenes.icosphere(3)
    cfg = RasterConfig.from_camera(capture_camera(s, "+z", 256))
    w = shard.fragment_weights(s, CaptureStrategy.normal_space(), cfg, 8)
    assert w.shape == (8 ** 8 // shard.tile_leaves(8),)
    assert w.sum() > s.n_triangles
    assert w is shard.fragment_weights(s, CaptureStrategy.normal_space(), cfg, 8)  # cached


def test_thread_comm_semantics():
    comms = shard.ThreadComm.group(3)
    out = [None] * 3

    def run(c):
        g = c.all_gather_int(10 + c.rank)
        t = torch.tensor([5 - c.rank, c.rank, -0.0 if c.rank else 2.5], dtype=torch.float64)
        mn = c.all_reduce_(t.clone(), "min")
        mx = c.all_reduce_(t.clone(), "max")
        sm = c.all_reduce_(t.clone(), "sum")
        out[c.rank] = (g, mn.tolist(), mx.tolist(), sm.tolist())

    th = [threading.Thread(target=run, args=(c,)) for c in comms]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r in range(3):
        g, mn, mx, sm = out[r]
        assert g == [10, 11, 12]
        assert mn == [3.0, 0.0, -0.0]
        assert mx == [5.0, 2.0, 2.5]
        assert sm == [12.0, 3.0, 2.5]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = shard.TorchComm()
        g = c.all_gather_int(1000 * (rank + 1))
        keys = torch.tensor([7 - rank, -(2 ** 62), 2 ** 63 - 1], dtype=torch.int64)
        c.all_reduce_(keys, "min")
        img = torch.tensor([-0.0, 0.25 * (rank + 1)], dtype=torch.float64)
        if rank == 0:
            img[0] = 0.75
        c.all_reduce_(img, "sum")
        pyr = torch.tensor([1 << rank, 0], dtype=torch.uint8)
        c.all_reduce_(pyr, "max")
        q.put((rank, g, keys.tolist(), img.tolist(), pyr.tolist()))
    finally:
        dist.destroy_process_group()


def test_torch_comm_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, g, keys, img, pyr in res:
        assert g == [1000, 2000]
        assert keys == [6, -(2 ** 62), 2 ** 63 - 1]
        assert img == [0.75, 0.75]
        assert pyr == [2, 0]
