"""CPU: the pipeline oracle (uniform noise + separable Gaussian smoothing,
SURVEY.md 8(f) rank 3) is bit-identical to the compiled reference
(datagen.hpp:57-62, 66-122), and rejects the widths the reference rejects."""
import numpy as np
import pytest

import oracle

ref_only = pytest.mark.skipif(not oracle.ref_available(), reason="reference not compiled here")

CASES = [((7, 9, 11), 2.0, 13), ((1, 1, 40), 4.0, 25), ((30, 1, 1), 1.5, 1), ((13, 17), 0.7, 3),
         ((5, 6, 7), 3.0, 7), ((16, 16, 16), 2.0, 13), ((3, 40, 2), 8.0, 31)]


@ref_only
@pytest.mark.parametrize("shape,sigma,width", CASES)
def test_smoothing_matches_reference_bitwise(shape, sigma, width):
    x = oracle.ref_uniform_noise(shape, 7)
    assert np.array_equal(x.view(np.uint32), oracle.uniform_noise(shape, 7).view(np.uint32))
    a = oracle.ref_gaussian_smooth(x, sigma, width)
    b = oracle.gaussian_smooth(x, sigma, width)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    # iterated, as bench_run does
    a2 = oracle.ref_gaussian_smooth(a, sigma, width)
    b2 = oracle.gaussian_smooth(b, sigma, width)
    assert np.array_equal(a2.view(np.uint32), b2.view(np.uint32))


@ref_only
@pytest.mark.parametrize("width", [0, 2, -3])
def test_invalid_widths(width):
    x = np.zeros((3, 3, 3), np.float32)
    with pytest.raises(ValueError, match="odd and >= 1"):
        oracle.ref_gaussian_smooth(x, 1.0, width)
    with pytest.raises(ValueError, match="odd and >= 1"):
        oracle.gaussian_smooth(x, 1.0, width)


@ref_only
def test_reference_bench_run_reports():
    r = oracle.ref_bench_run((16, 16, 16), 2)
    assert r["total_s"] > 0 and r["ecc_avg_s"] > 0 and r["smooth_avg_s"] > 0
