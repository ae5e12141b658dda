"""GPU parity of the bit-sliced 2D u8 kernel (k_u8_2d.cu) against the oracle.

The kernel serves single 2D u8 images (w2 == 1): a warp holds 32 chunks of 32
pixels of a row (lanes 0 / 31 are halo, 960 owned pixels per strip) and
sweeps a band of rows; rows that are not a multiple of 16 bytes are first
copied to a 16-byte pitch.  The cases target strip and chunk edges, band
splits, ties around 255 (the collar value), slabs, the fused single-launch
curve and the full paper-size images.  Bit-exact.
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
    (1, 16), (1, 1), (2, 1), (7, 3), (5, 31), (9, 32), (3, 33), (40, 64), (33, 959), (17, 960),
    (21, 961), (12, 1920), (11, 1921), (64, 2000), (100, 4097), (257, 255), (1000, 48),
    (3000, 16), (2, 30 * 32 * 3 + 5),
])
def test_random_shapes(ctx, shape):
    rng = np.random.default_rng(sum(shape) + 7)
    _check(ctx, rng.integers(0, 256, shape).astype(np.uint8))


@pytest.mark.parametrize("lo,hi", [(250, 256), (0, 2), (254, 256), (100, 104)])
def test_ties_and_collar_values(ctx, lo, hi):
    rng = np.random.default_rng(lo + 1)
    for shape in [(37, 1024), (64, 961), (5, 96), (300, 33)]:
        _check(ctx, rng.integers(lo, hi, shape).astype(np.uint8))


def test_constant_plateau_and_stripes(ctx):
    for val in (0, 255, 77):
        img = np.full((130, 2049), val, np.uint8)
        a = ctx.vcec(img)
        assert list(a.values) == [val] and list(a.changes) == [1]
    y, x = np.meshgrid(np.arange(333), np.arange(1500), indexing="ij")
    _check(ctx, (((x >> 3) + (y >> 3)) & 255).astype(np.uint8))
    _check(ctx, ((x % 2) * 255).astype(np.uint8))        # columns alternate 0 / 255
    _check(ctx, ((y % 2) * 255).astype(np.uint8))        # rows alternate
    _check(ctx, (((x + y) % 2) * 200).astype(np.uint8))  # checkerboard


def test_streamed_chunks_and_misaligned_views(ctx):
    import torch
    rng = np.random.default_rng(21)
    img = rng.integers(0, 256, (517, 1000)).astype(np.uint8)
    want = oracle.vcec(img)
    for c in (1, 2, 3, 7, 517):
        plan = eb.plan_chunks(eb.Dims.of(img.shape), eb.ChunkTarget.count(c))
        got = eb.process_image(img, plan)
        assert np.array_equal(got.changes, want[1]), c
    flat = torch.empty(img.size + 3, dtype=torch.uint8, device="cuda")
    flat[3:].copy_(torch.from_numpy(img.ravel()))
    got = ctx.vcec(flat[3:].view(img.shape))
    assert np.array_equal(got.changes, want[1])


def test_slabs_match_whole(ctx):
    import torch
    rng = np.random.default_rng(12)
    img = rng.integers(0, 256, (300, 1024)).astype(np.uint8)
    want = oracle.vcec(img)
    dev = torch.from_numpy(img).cuda()
    hist = torch.zeros(512, dtype=torch.int64, device="cuda")
    dims = eb.Dims.of(img.shape)
    for own0, own1 in [(0, 1), (1, 100), (100, 101), (101, 299), (299, 300)]:
        p0, p1 = max(own0 - 1, 0), min(own1 + 1, 300)
        ctx.accumulate_slab(dev[p0:p1].contiguous(), dims, p0, own0, own1, hist)
    torch.cuda.synchronize()
    h = hist.cpu().numpy()
    bins = np.nonzero(h[256:])[0]
    assert np.array_equal(bins, want[0].astype(np.int64))
    assert np.array_equal(h[bins], want[1])


def _device_curve(ctx, dev):
    import torch
    bins = torch.empty(256, dtype=torch.int32, device="cuda")
    chg = torch.empty(256, dtype=torch.int64, device="cuda")
    chi = torch.empty(256, dtype=torch.int64, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    ctx.curve_device(dev, eb.Dims.of(tuple(dev.shape)), bins, chg, chi, cnt)
    torch.cuda.synchronize()
    m = int(cnt.item())
    return bins[:m].cpu().numpy(), chg[:m].cpu().numpy(), chi[:m].cpu().numpy()


def test_fused_single_launch_repeats(ctx):
    """ecc_curve_device: one launch with the last-CTA K3; the workspace resets
    itself, so back-to-back calls on different images stay exact."""
    import torch
    rng = np.random.default_rng(5)
    for shape in [(256, 256), (1, 5000), (4096, 17), (700, 3000)]:
        img = rng.integers(0, 256, shape).astype(np.uint8)
        v, c = oracle.vcec(img)
        for _ in range(2):
            b, ch, chi = _device_curve(ctx, torch.from_numpy(img).cuda())
            assert np.array_equal(b, v.astype(np.int32)) and np.array_equal(ch, c)
            assert np.array_equal(chi, np.cumsum(c))


@pytest.mark.parametrize("shape", [(8192, 8192), (6400, 3200)])
def test_paper_size_images(ctx, shape):
    """The paper's 2D sizes (8192^2 Gaussian random field, 6400 x 3200 map)
    as random u8 images, against the C oracle."""
    import torch
    dev = torch.empty(shape, dtype=torch.uint8, device="cuda")
    ctx.fill_synthetic(dev, seed=3)
    img = dev.cpu().numpy()
    v, c = oracle.vcec(img)
    b, ch, chi = _device_curve(ctx, dev)
    assert np.array_equal(b, v.astype(np.int32)) and np.array_equal(ch, c)
    assert int(chi[-1]) == 1


def test_cluster_path_interleaved_with_large_images(ctx):
    """Small images run in one thread-block cluster whose CTA 0 reduces the
    histogram over distributed shared memory (fin_u8.cuh, cluster_finalize)
    and never touches the fused global histogram or ticket; larger images use
    the global-atomics path.  Alternate the two (bands of 1..4 rows and the
    band-5 boundary at 1025 x 256) and check every curve."""
    rng = np.random.default_rng(23)
    shapes = [(256, 256), (1500, 1500), (512, 512), (1024, 256), (1025, 256), (3, 1000),
              (2048, 300), (300, 1000), (1, 5000), (767, 511)]
    for shape in shapes + shapes[::-1]:
        img = rng.integers(0, 256, shape).astype(np.uint8)
        _check(ctx, img)
        # the device-resident single-launch curve as well
        import torch
        d = torch.from_numpy(img).cuda()
        bins = torch.empty(256, dtype=torch.int32, device="cuda")
        chg = torch.empty(256, dtype=torch.int64, device="cuda")
        chi = torch.empty(256, dtype=torch.int64, device="cuda")
        cnt = torch.empty(1, dtype=torch.int64, device="cuda")
        ctx.curve_device(d, eb.Dims(shape[0], shape[1], 1), bins, chg, chi, cnt)
        torch.cuda.synchronize()
        v, c = oracle.vcec(img)
        m = int(cnt.item())
        assert m == len(v), shape
        assert np.array_equal(bins[:m].cpu().numpy().astype(np.int64), v.astype(np.int64)), shape
        assert np.array_equal(chg[:m].cpu().numpy(), c), shape
        assert np.array_equal(chi[:m].cpu().numpy(), np.cumsum(c)), shape


@pytest.mark.parametrize("w", [1, 31, 32, 33, 64, 96, 128, 160, 256, 480, 512])
def test_packed_rows(ctx, w):
    """Rows of <= 16 chunks run packed, 32 / L rows per warp (L lanes a row,
    L a power of two >= the chunk count; the last lane of a full group has
    the row's right collar as its neighbour).  Heights leave the last warp's
    row groups partly empty; both the single-launch curve (small images: the
    cluster path) and slab accumulation (the regular grid) are checked."""
    import torch
    rng = np.random.default_rng(w)
    for h in (1, 2, 3, 5, 33, 257, 1031):
        img = rng.integers(0, 256, (h, w)).astype(np.uint8)
        if h % 2:
            img[:, :: max(1, w // 3)] = 255  # ties with the collar value
        _check(ctx, img)
        want = oracle.vcec(img)
        dev = torch.from_numpy(img).cuda()
        hist = torch.zeros(512, dtype=torch.int64, device="cuda")
        dims = eb.Dims.of(img.shape)
        cut = h // 2
        for own0, own1 in [(0, cut), (cut, h)]:
            if own1 > own0:
                p0, p1 = max(own0 - 1, 0), min(own1 + 1, h)
                ctx.accumulate_slab(dev[p0:p1].contiguous(), dims, p0, own0, own1, hist)
        torch.cuda.synchronize()
        hh = hist.cpu().numpy()
        bins = np.nonzero(hh[256:])[0]
        assert np.array_equal(bins, want[0].astype(np.int64)), (h, w)
        assert np.array_equal(hh[bins], want[1]), (h, w)
