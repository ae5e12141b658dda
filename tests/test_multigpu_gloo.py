"""The N > 1 path on CPU: world_size-2 (and 3) process groups over gloo run
the same sharding driver bench.py runs over NCCL (paper_2203_09087_b200/
shard.py): balanced z-slabs with halo planes, one all_reduce(sum) of the
int64 histogram, then compaction + prefix sum.  The per-slab accumulate is
played by the oracle (test infrastructure), so what is tested here is the
host logic: bounds, halos, the single exchange and rank invariance."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2203_09087_b200.shard import Shard, shard_bounds, sharded_histogram


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slab_hist(img, shard: Shard, nbins):
    """Histogram of the owned planes computed from the slab + halo planes
    only (what a rank's GPU sees): changes of the held planes, owned part."""
    held = np.ascontiguousarray(img[shard.plane0:shard.plane1])
    ch = oracle.changes(held).reshape(held.shape[0], -1)
    # the held block's own collar is wrong at the slab cut, except where the
    # cut is the image boundary; keep only owned planes, which see true data
    lo = shard.own0 - shard.plane0
    own_ch = ch[lo:lo + (shard.own1 - shard.own0)]
    own_v = held[lo:lo + (shard.own1 - shard.own0)].reshape(own_ch.shape[0], -1)
    h = np.zeros(2 * nbins, np.int64)
    np.add.at(h, own_v.ravel().astype(np.int64), own_ch.ravel().astype(np.int64))
    np.add.at(h, nbins + own_v.ravel().astype(np.int64), 1)
    return h


def _worker(rank, world, port, img, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nbins = 256 if img.dtype == np.uint8 else 65536
    sh = shard_bounds(img.shape[0], world, rank)
    hist = torch.zeros(2 * nbins, dtype=torch.int64)

    def accumulate(shard, h):
        h += torch.from_numpy(_slab_hist(img, shard, nbins))

    sharded_histogram(sh, accumulate, hist, dist.all_reduce)
    h = hist.numpy()
    occ = np.nonzero(h[nbins:])[0]
    q.put((rank, occ, h[occ], np.cumsum(h[occ])))
    dist.destroy_process_group()


def _run(world, img):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, img, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_curve_equals_whole_volume(world):
    rng = np.random.default_rng(world)
    img = rng.integers(0, 256, (11, 13, 9)).astype(np.uint8)
    v, c = oracle.vcec(img)
    for rank, occ, ch, chi in _run(world, img):
        assert np.array_equal(occ, v.astype(np.int64)), rank
        assert np.array_equal(ch, c), rank
        assert chi[-1] == 1


def test_gloo_u16_and_more_ranks_than_planes():
    rng = np.random.default_rng(5)
    img = rng.integers(0, 9, (2, 7, 5)).astype(np.uint16)
    v, c = oracle.vcec(img)
    for rank, occ, ch, chi in _run(3, img):  # rank 2 owns nothing
        assert np.array_equal(occ, v.astype(np.int64)) and np.array_equal(ch, c)


def test_shard_bounds_cover_and_balance():
    for w0 in (1, 2, 7, 64, 1000, 4096):
        for world in (1, 2, 3, 4, 8):
            shards = [shard_bounds(w0, world, r) for r in range(world)]
            assert shards[0].own0 == 0 and shards[-1].own1 == w0
            for a, b in zip(shards, shards[1:]):
                assert a.own1 == b.own0
            sizes = [s.own1 - s.own0 for s in shards]
            assert max(sizes) - min(sizes) <= 1
            for s in shards:
                if s.own1 > s.own0:
                    assert s.plane0 == max(s.own0 - 1, 0) and s.plane1 == min(s.own1 + 1, w0)
    # BASELINE shapes divide evenly
    assert all(shard_bounds(1024, 8, r).own1 - shard_bounds(1024, 8, r).own0 == 128 for r in range(8))
