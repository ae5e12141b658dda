"""GPU: the GPU-resident pipeline -- uniform noise,
Gaussian smoothing and bench_run -- bit-identical to the oracle (which
tests/test_pipeline_oracle.py pins to the reference)."""
import numpy as np
import pytest

import oracle
import paper_2203_09087_b200 as eb

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("shape,sigma,width", [
    ((7, 9, 11), 2.0, 13), ((1, 1, 40), 4.0, 25), ((30, 1, 1), 1.5, 1), ((13, 17), 0.7, 3),
    ((5, 6, 7), 3.0, 7), ((64, 48, 80), 2.0, 13), ((3, 40, 2), 8.0, 31), ((100, 300), 4.0, 25)])
def test_noise_and_smoothing_bitwise(ctx, shape, sigma, width):
    import torch
    x = torch.empty(shape, dtype=torch.float32, device="cuda")
    ctx.uniform_noise(x, seed=11)
    torch.cuda.synchronize()
    want = oracle.uniform_noise(shape, 11)
    assert np.array_equal(_bits(x.cpu().numpy()), _bits(want))
    y = ctx.gaussian_smooth(x, sigma, width)
    torch.cuda.synchronize()
    ws = oracle.gaussian_smooth(want, sigma, width)
    assert np.array_equal(_bits(y.cpu().numpy()), _bits(ws))
    ctx.gaussian_smooth(y, sigma, width, out=y)  # in place, iterated
    torch.cuda.synchronize()
    assert np.array_equal(_bits(y.cpu().numpy()), _bits(oracle.gaussian_smooth(ws, sigma, width)))


def test_invalid_width_is_rejected(ctx):
    import torch
    x = torch.zeros((4, 4, 4), dtype=torch.float32, device="cuda")
    with pytest.raises(eb.EccError, match="odd and >= 1"):
        ctx.gaussian_smooth(x, 1.0, 4)
    with pytest.raises(eb.EccError, match="at least one iteration"):
        ctx.bench_run(eb.Dims(4, 4, 4), 0)


@pytest.mark.parametrize("shape,iters", [((24, 30, 36), 2), ((40, 40, 1), 3), ((16, 16, 16), 1)])
def test_bench_run_curve_matches_oracle_pipeline(ctx, shape, iters):
    """The last iteration's curve (point count, first and last chi) equals
    the oracle's ECC of the oracle's iterated smoothing of the same noise."""
    rep = ctx.bench_run(eb.Dims(*shape), iters, seed=1, sigma=2.0, width=13)
    x = oracle.uniform_noise(shape, 1)
    for _ in range(iters):
        x = oracle.gaussian_smooth(x, 2.0, 13)
    v, c = oracle.vcec(x)
    chi = np.cumsum(c)
    assert rep.iterations == iters and rep.voxels == int(np.prod(shape))
    assert rep.last_points == len(v)
    assert rep.last_chi_first == chi[0] and rep.last_chi_last == chi[-1] == 1
    assert rep.ecc_avg_s > 0 and rep.smooth_avg_s > 0 and rep.total_s > 0


def test_smoothed_volume_curve_full(ctx):
    """Full curve of a device-smoothed volume through the exact f32 path."""
    import torch
    shape = (48, 40, 56)
    x = torch.empty(shape, dtype=torch.float32, device="cuda")
    ctx.uniform_noise(x, seed=3)
    y = ctx.gaussian_smooth(x, 2.0, 13)
    torch.cuda.synchronize()
    got = ctx.vcec(y)
    v, c = oracle.vcec(oracle.gaussian_smooth(oracle.uniform_noise(shape, 3), 2.0, 13))
    assert np.array_equal(_bits(got.values), _bits(v)) and np.array_equal(got.changes, c)
