"""GPU parity of the column layouts of the bit-sliced 3D kernels (k_u8_3d.cu,
k_u16_3d.cu) against the oracle, bit-exact.

Columns are 32 lanes (axis 1) x 32 bits (axis 2).  Interior columns own 30
of each, the first and last own 31 with a *virtual* collar (no lane / bit
holds the voxel beyond the image edge; bits.cuh cols): the widths below sit
on the boundaries of that layout (31 / 32 / 33 = one column or two, 62 / 63
= two or three, 92 / 93, 512 = 31 + 15 x 30 + 31) along both in-plane axes,
with values near 255 / 65535 so that ties against the collar sentinel are
frequent.  k_u16_3d uses the virtual-collar instantiation only where it
saves columns, so both of its layouts are hit.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

W1S = [31, 32, 33, 62, 63, 92, 93]
W2S_U8 = [32, 48, 64, 96]          # the u8 fast path wants rows of 16 bytes
W2S_U16 = [32, 40, 64, 96, 120]    # u16: rows of 8 elements


def _check(ctx, img):
    a = ctx.vcec(img)
    v, c = oracle.vcec(img)
    assert np.array_equal(a.values.astype(np.int64), v.astype(np.int64)), img.shape
    assert np.array_equal(a.changes, c), img.shape


@pytest.mark.parametrize("w1", W1S)
def test_u8_column_edges(ctx, w1):
    rng = np.random.default_rng(w1)
    for w2 in W2S_U8:
        _check(ctx, rng.integers(0, 256, (5, w1, w2)).astype(np.uint8))
        _check(ctx, rng.integers(252, 256, (4, w1, w2)).astype(np.uint8))


@pytest.mark.parametrize("w1", W1S)
def test_u16_column_edges(ctx, w1):
    rng = np.random.default_rng(100 + w1)
    for w2 in W2S_U16:
        _check(ctx, rng.integers(0, 65536, (5, w1, w2)).astype(np.uint16))
        _check(ctx, rng.integers(65532, 65536, (4, w1, w2)).astype(np.uint16))


@pytest.mark.parametrize("dtype,hi", [(np.uint8, 256), (np.uint16, 65536)])
def test_512_wide_planes(ctx, dtype, hi):
    # 17 columns per axis (the C2 layout), ties near the sentinel on the edges
    rng = np.random.default_rng(7)
    img = rng.integers(0, hi, (6, 512, 512)).astype(dtype)
    img[:, :2, :] = hi - 1
    img[:, :, -2:] = hi - 1
    _check(ctx, img)
