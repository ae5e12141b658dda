"""GPU parity of the 16-bit 2D kernel (k_u16_2d.cu) against the oracle.

Single 2D u16 images, and affine-quantised f32 images (mapped to u16 bin
indices first), run the bit-sliced 16-plane stencil with the packed 65536-bin
shared-memory histogram, one CTA per SM.  Cases: strip / chunk edges, odd
widths (padded pitch), ties at 0xFFFF (the collar value), slabs, the spill
path (many isolated minima on one value) and the paper-size image.
Bit-exact.
"""
import numpy as np
import pytest

import oracle
import paper_2203_09087_b200 as eb

pytestmark = pytest.mark.gpu


def _check(ctx, img, binmap=None):
    a = ctx.vcec(img, binmap=binmap) if binmap else ctx.vcec(img)
    v, c = oracle.vcec(img)
    if img.dtype == np.float32:
        assert np.array_equal(np.asarray(a.values, np.float32).view(np.uint32),
                              np.asarray(v, np.float32).view(np.uint32)), img.shape
    else:
        assert np.array_equal(a.values.astype(np.int64), v.astype(np.int64)), img.shape
    assert np.array_equal(a.changes, c), img.shape


@pytest.mark.parametrize("shape", [
    (1, 8), (1, 1), (3, 1), (7, 3), (5, 31), (9, 32), (3, 33), (40, 64), (33, 959), (17, 960),
    (21, 961), (12, 1920), (64, 2000), (100, 4097), (257, 255), (2000, 24),
])
def test_random_shapes_u16(ctx, shape):
    rng = np.random.default_rng(sum(shape) + 17)
    _check(ctx, rng.integers(0, 65536, shape).astype(np.uint16))


@pytest.mark.parametrize("lo,hi", [(65530, 65536), (0, 2), (1000, 1004)])
def test_ties_and_collar_values(ctx, lo, hi):
    rng = np.random.default_rng(lo + 3)
    for shape in [(37, 1024), (64, 961), (300, 33)]:
        _check(ctx, rng.integers(lo, hi, shape).astype(np.uint16))


def test_affine_f32(ctx):
    rng = np.random.default_rng(8)
    for shape in [(300, 1000), (77, 65), (1, 5000)]:
        q = (rng.integers(0, 65536, shape) * 2.0 ** -16).astype(np.float32)
        _check(ctx, q, binmap=eb.quantised_binmap(65536))
    q = (rng.integers(0, 1000, (129, 513)) * 0.25).astype(np.float32)
    _check(ctx, q, binmap=eb.quantised_binmap(1000, 0.0, 250.0))
    bad = (rng.integers(0, 65536, (64, 64)) * 2.0 ** -16).astype(np.float32)
    bad[5, 7] = 0.3
    with pytest.raises(eb.EccError) as ei:
        ctx.vcec(bad, binmap=eb.quantised_binmap(65536))
    assert ei.value.code == eb.ECC_EBINMAP


def test_streamed_chunks_and_slabs(ctx):
    rng = np.random.default_rng(22)
    img = rng.integers(0, 65536, (517, 1000)).astype(np.uint16)
    want = oracle.vcec(img)
    for c in (1, 2, 5, 517):
        plan = eb.plan_chunks(eb.Dims.of(img.shape), eb.ChunkTarget.count(c), np.uint16)
        got = eb.process_image(img, plan)
        assert np.array_equal(got.changes, want[1]), c


def test_spill_path_isolated_minima(ctx):
    """4096^2 with every other pixel of every other row = 0: 4M isolated
    minima on one bin, so its 16-bit half crosses the band many times in
    every CTA and the exact spill path runs."""
    rng = np.random.default_rng(23)
    img = rng.integers(1000, 60000, (4096, 4096)).astype(np.uint16)
    img[::2, ::2] = 0
    _check(ctx, img)


def test_paper_size_image(ctx):
    import torch
    dev = torch.empty((8192, 8192), dtype=torch.uint16, device="cuda")
    ctx.fill_synthetic(dev, seed=5)
    img = dev.cpu().numpy()
    got = ctx.vcec(dev)
    v, c = oracle.vcec(img)
    assert np.array_equal(got.values.astype(np.int64), v.astype(np.int64))
    assert np.array_equal(got.changes, c)
