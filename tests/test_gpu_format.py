"""GPU: batched curve files (ecc_batch_format) are
byte-identical to the reference writer (write_curve, curve.hpp:87-121):
against the compiled reference for CSV where it is available, and against a
line-for-line Python restatement of the same layout for CSV and JSON."""
import numpy as np
import pytest

import oracle
import paper_2203_09087_b200 as eb

pytestmark = pytest.mark.gpu


def _csv(t, chi):
    return ("threshold,euler_characteristic\n" +
            "".join(f"{int(a)},{int(b)}\n" for a, b in zip(t, chi))).encode()


def _json(t, chi):
    return ("[" + ",".join(f'{{"t":{int(a)},"chi":{int(b)}}}' for a, b in zip(t, chi)) +
            "]\n").encode()


@pytest.mark.parametrize("dt,hi,shape", [(np.uint8, 256, (7, 33, 45)), (np.uint16, 65536, (5, 64, 80)),
                                          (np.uint16, 40, (3, 20, 30)), (np.uint8, 3, (4, 9, 9))])
def test_batch_format_matches_writer(ctx, dt, hi, shape):
    import torch
    rng = np.random.default_rng(hi)
    imgs = rng.integers(0, hi, shape).astype(dt)
    dev = torch.from_numpy(imgs).cuda()
    chi, pres = ctx.batch2d(dev)
    torch.cuda.synchronize()
    csv = ctx.batch_format(chi, pres, dt, "csv")
    js = ctx.batch_format(chi, pres, dt, "json")
    chi_h, pres_h = chi.cpu().numpy(), pres.cpu().numpy().view(np.uint32)
    for b in range(shape[0]):
        t, c = eb.curve_batch_to_points(chi_h[b], pres_h[b])
        assert csv[b] == _csv(t, c), b
        assert js[b] == _json(t, c), b
        v, ch = oracle.vcec(imgs[b])
        assert np.array_equal(t, v.astype(np.int64)) and np.array_equal(c, np.cumsum(ch))
        if oracle.ref_available():
            assert csv[b] == oracle.ref_csv(v, np.cumsum(ch))


def test_batch_format_c3_scale(ctx):
    """4096 x 512^2 u16 (BASELINE config 3): every image's CSV is sized and
    written on the device; spot-check images 0 and 4095 against the
    Appendix-B golden digests through the reference's CSV hash."""
    import torch
    imgs = torch.empty((4096, 512, 512), dtype=torch.uint16, device="cuda")
    ctx.fill_synthetic(imgs, seed=1)
    chi, pres = ctx.batch2d(imgs)
    torch.cuda.synchronize()
    files = ctx.batch_format(chi, pres, np.uint16, "csv")
    assert len(files) == 4096
    import hashlib, json, os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))["configs"]
    for b in (0, 4095):
        t, c = eb.curve_batch_to_points(chi[b].cpu().numpy(), pres[b].cpu().numpy().view(np.uint32))
        assert files[b] == _csv(t, c)
        assert oracle.curve_digest(t, c) == gold[f"C3_{b}"]["digest"]


def _zero_crossings(t, chi):
    out = []
    for i in range(len(t)):
        if chi[i] == 0:
            out.append(int(t[i]))
        elif i > 0 and chi[i - 1] != 0 and (chi[i] > 0) != (chi[i - 1] > 0):
            out.append(int(t[i]))
    return out


@pytest.mark.parametrize("dt,hi,shape", [(np.uint8, 256, (9, 40, 40)), (np.uint16, 65536, (4, 96, 96)),
                                          (np.uint16, 300, (6, 50, 70)), (np.uint8, 6, (5, 12, 12))])
def test_batch_zero_crossings(ctx, dt, hi, shape):
    """zero_crossings (curve.hpp:36-50) on the device == its restatement."""
    import torch
    rng = np.random.default_rng(hi + 1)
    imgs = rng.integers(0, hi, shape).astype(dt)
    chi, pres = ctx.batch2d(torch.from_numpy(imgs).cuda())
    zc = ctx.batch_zero_crossings(chi, pres, dt)
    torch.cuda.synchronize()
    chi_h, pres_h, zc_h = chi.cpu().numpy(), pres.cpu().numpy().view(np.uint32), zc.cpu().numpy().view(np.uint32)
    for b in range(shape[0]):
        t, c = eb.curve_batch_to_points(chi_h[b], pres_h[b])
        bits = np.unpackbits(zc_h[b].view(np.uint8), bitorder="little").astype(bool)
        assert list(np.nonzero(bits)[0]) == _zero_crossings(t, c), b
