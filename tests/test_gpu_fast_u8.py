"""GPU parity of the bit-sliced 3D u8 kernel (k_u8_3d.cu) against the oracle.

The kernel serves 3D u8 volumes whose axis-2 rows are a multiple of 16
bytes; it tiles axes 1/2 into columns of 30 (31 at the image edges: virtual
collar, tests/test_gpu_columns.py) with a 1-voxel halo and splits the
(column, plane) work evenly over warps, so the cases below target column
edges, uneven splits, tiny dims, slabs, ties around 255 (the collar value)
and constant / plateau inputs.  Bit-exact.
"""
import numpy as np
import pytest

import oracle
import paper_2203_09087_b200 as eb

pytestmark = pytest.mark.gpu


def _check(ctx, img):
    a = ctx.vcec(img)
    v, c = oracle.vcec(img)
    assert np.array_equal(a.values.astype(np.int64), v.astype(np.int64)), img.shape
    assert np.array_equal(a.changes, c), img.shape


@pytest.mark.parametrize("shape", [
    (1, 1, 16), (1, 2, 16), (2, 1, 32), (3, 30, 32), (4, 31, 16), (5, 32, 48), (7, 61, 64),
    (9, 60, 96), (33, 29, 32), (17, 90, 128), (64, 64, 64), (40, 100, 160), (2, 512, 512),
    (31, 17, 240), (8, 3, 496),
])
def test_random_shapes(ctx, shape):
    rng = np.random.default_rng(sum(shape))
    _check(ctx, rng.integers(0, 256, shape).astype(np.uint8))


@pytest.mark.parametrize("lo,hi", [(250, 256), (0, 2), (254, 256), (100, 104)])
def test_ties_and_collar_values(ctx, lo, hi):
    # many ties, and values equal to the 255 the kernel uses for the collar
    rng = np.random.default_rng(lo)
    for shape in [(6, 35, 48), (12, 62, 32), (3, 5, 16)]:
        _check(ctx, rng.integers(lo, hi, shape).astype(np.uint8))


def test_constant_and_plateau(ctx):
    for val in (0, 255, 77):
        img = np.full((13, 47, 64), val, np.uint8)
        a = ctx.vcec(img)
        assert list(a.values) == [val] and list(a.changes) == [1]
    z, y, x = np.meshgrid(np.arange(40), np.arange(70), np.arange(96), indexing="ij")
    img = (((x >> 3) + (y >> 3) + (z >> 3)) & 255).astype(np.uint8)
    _check(ctx, img)
    # large constant run: exercises the histogram drain (>5000 voxels per bin)
    img = np.full((64, 128, 128), 9, np.uint8)
    img[::7, ::5, ::3] = 200
    _check(ctx, img)


def test_slabs_match_whole(ctx):
    """ecc_accumulate_slab over z-slabs with halo planes sums to the whole."""
    import torch
    rng = np.random.default_rng(11)
    img = rng.integers(0, 256, (50, 70, 80)).astype(np.uint8)
    want = oracle.vcec(img)
    dev = torch.from_numpy(img).cuda()
    hist = torch.zeros(512, dtype=torch.int64, device="cuda")
    dims = eb.Dims.of(img.shape)
    for own0, own1 in [(0, 1), (1, 17), (17, 18), (18, 49), (49, 50)]:
        p0, p1 = max(own0 - 1, 0), min(own1 + 1, 50)
        ctx.accumulate_slab(dev[p0:p1].contiguous(), dims, p0, own0, own1, hist)
    torch.cuda.synchronize()
    h = hist.cpu().numpy()
    bins = np.nonzero(h[256:])[0]
    assert np.array_equal(bins, want[0].astype(np.int64))
    assert np.array_equal(h[bins], want[1])


def test_config2_size_properties(ctx, golden):
    """Full C2 size: chi ends at 1, first point and the golden curve digest."""
    import torch
    dev = torch.empty((512, 512, 512), dtype=torch.uint8, device="cuda")
    ctx.fill_synthetic(dev, seed=1)
    torch.cuda.synchronize()
    cur = ctx.curve(dev)
    assert int(cur.chi[-1]) == 1 and cur.size() == 256
    assert int(cur.chi[0]) == 499566
    assert oracle.curve_digest(cur.thresholds, cur.chi) == golden["configs"]["C2"]["digest"]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sharded_driver_on_one_gpu(ctx, world):
    """bench.py's N-rank step with the ranks run one after another on one GPU
    (the all-reduce becomes a running sum): every rank count gives the same
    curve, equal to the oracle's."""
    import torch
    from paper_2203_09087_b200.shard import shard_bounds, sharded_histogram
    rng = np.random.default_rng(world)
    img = rng.integers(0, 256, (37, 64, 96)).astype(np.uint8)
    dims = eb.Dims.of(img.shape)
    total = torch.zeros(512, dtype=torch.int64, device="cuda")
    for r in range(world):
        sh = shard_bounds(img.shape[0], world, r)
        slab = torch.from_numpy(np.ascontiguousarray(img[sh.plane0:sh.plane1])).cuda()
        h = torch.zeros(512, dtype=torch.int64, device="cuda")
        sharded_histogram(sh, lambda s, hh: ctx.accumulate_slab(slab, dims, s.plane0, s.own0,
                                                                 s.own1, hh), h,
                          lambda hh: (torch.cuda.synchronize(), total.add_(hh)))
    bins = torch.empty(256, dtype=torch.int32, device="cuda")
    chg = torch.empty(256, dtype=torch.int64, device="cuda")
    chi = torch.empty(256, dtype=torch.int64, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    ctx.finalize(total, 256, bins, chg, chi, cnt)
    torch.cuda.synchronize()
    m = int(cnt.item())
    v, c = oracle.vcec(img)
    assert np.array_equal(bins[:m].cpu().numpy(), v.astype(np.int32))
    assert np.array_equal(chg[:m].cpu().numpy(), c)
    assert np.array_equal(chi[:m].cpu().numpy(), np.cumsum(c))


@pytest.mark.parametrize("shape", [(40, 50, 77), (9, 33, 100), (5, 7, 3), (3, 300, 17), (17, 16, 129)])
def test_odd_row_widths_take_the_padded_fast_path(ctx, shape):
    """Rows that are not a multiple of 16 bytes (or a misaligned base) are
    copied once into a 16-byte row pitch and run through the TMA kernel."""
    import torch
    rng = np.random.default_rng(sum(shape) + 1)
    img = rng.integers(0, 256, shape).astype(np.uint8)
    _check(ctx, img)
    # misaligned device base: a view starting one byte into a buffer
    flat = torch.empty(img.size + 1, dtype=torch.uint8, device="cuda")
    flat[1:].copy_(torch.from_numpy(img.ravel()))
    dev = flat[1:].view(shape)
    got = ctx.vcec(dev)
    v, c = oracle.vcec(img)
    assert np.array_equal(got.changes, c)


@pytest.mark.parametrize("shape", [(256, 512, 512), (130, 512, 512), (67, 700, 768)])
def test_overlapped_host_input(ctx, shape):
    """Large host u8 volumes take the overlapped path of ecc_vcec / ecc_curve
    (chunked H2D on the copy stream, each chunk's kernel as soon as it and
    its halo plane have landed); the curve equals the oracle's."""
    rng = np.random.default_rng(sum(shape))
    img = rng.integers(0, 256, shape, dtype=np.uint8)
    _check(ctx, img)
    c = ctx.curve(img)
    assert int(c.chi[-1]) == 1


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_host_streaming(ctx, world):
    """ecc_accumulate_host (C5 on several GPUs): each "rank" streams only its
    planes + halos from its own host buffer, chunk by chunk; the summed
    histograms finalize to the oracle's curve (u8 and u16)."""
    import torch
    from paper_2203_09087_b200.shard import shard_bounds
    rng = np.random.default_rng(40 + world)
    for dt, hi, nb in ((np.uint8, 256, 256), (np.uint16, 65536, 65536)):
        img = rng.integers(0, hi, (45, 40, 48), dtype=dt)
        dims = eb.Dims.of(img.shape)
        total = torch.zeros(2 * nb, dtype=torch.int64, device="cuda")
        for r in range(world):
            sh = shard_bounds(img.shape[0], world, r)
            mine = np.ascontiguousarray(img[sh.plane0:sh.plane1])
            n = sh.own1 - sh.own0
            bounds = sorted({sh.own0 + n * k // 3 for k in range(4)})
            h = torch.zeros(2 * nb, dtype=torch.int64, device="cuda")
            ctx.accumulate_host(mine, sh.plane0, dims, bounds, h)
            total += h
        bins = torch.empty(nb, dtype=torch.int32, device="cuda")
        chg = torch.empty(nb, dtype=torch.int64, device="cuda")
        chi = torch.empty(nb, dtype=torch.int64, device="cuda")
        cnt = torch.empty(1, dtype=torch.int64, device="cuda")
        ctx.finalize(total, nb, bins, chg, chi, cnt)
        torch.cuda.synchronize()
        m = int(cnt.item())
        v, c = oracle.vcec(img)
        assert np.array_equal(bins[:m].cpu().numpy().astype(np.int64), v.astype(np.int64))
        assert np.array_equal(chg[:m].cpu().numpy(), c)
    # a chunk whose halo is not in the buffer is refused
    with pytest.raises(eb.EccError, match="host buffer holds"):
        ctx.accumulate_host(np.zeros((5, 40, 48), np.uint8), 10, eb.Dims(45, 40, 48), [10, 15],
                            torch.zeros(512, dtype=torch.int64, device="cuda"))


def test_fused_rank_exchange_two_processes():
    """ecc_curve_sharded across 2 processes (torchrun; CUDA IPC between them,
    on one GPU here, one GPU per rank in production): the histogram exchange
    fused into the launch gives every rank the oracle's curve, 3 volumes x 3
    consecutive steps (both exchange parities)."""
    import subprocess
    import sys as _sys
    root = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
    import socket
    with socket.socket() as so:  # a free port for the rendezvous
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    r = subprocess.run([_sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        __import__("os").path.join(root, "tools", "xchg_check.py")],
                       capture_output=True, text=True, timeout=300)
    assert "XCHG OK 2 ranks" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
