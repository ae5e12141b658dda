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


def _ref_writer_py(t, chi, fmt):
    """The reference layouts with the thresholds as the reference formats
    them (oracle.ref_csv for CSV when the reference is compiled)."""
    import oracle as o
    def tx(v):
        if np.issubdtype(np.asarray(t).dtype, np.floating):
            return repr_float(v)
        return str(int(v))
    if fmt == "vcec":
        return ("value,change\n" + "".join(f"{tx(a)},{int(b)}\n" for a, b in zip(t, chi))).encode()
    if fmt == "json":
        return ("[" + ",".join(f'{{"t":{tx(a)},"chi":{int(b)}}}' for a, b in zip(t, chi)) + "]\n").encode()
    return ("threshold,euler_characteristic\n" +
            "".join(f"{tx(a)},{int(b)}\n" for a, b in zip(t, chi))).encode()


def repr_float(v):
    """std::to_chars(float) text through the reference's own CSV writer (one
    point), which is the ground truth for the layout and the digits."""
    line = oracle.ref_csv(np.array([v], np.float32), np.array([0], np.int64)).decode()
    return line.split("\n")[1].split(",")[0]


@pytest.mark.parametrize("fmt", ["csv", "json", "vcec"])
def test_format_curve_f32_matches_reference_writer(ctx, fmt):
    """One f32 curve formatted on the GPU (ecc_format_curve; f2s.cuh is the
    shortest round-trip formatter) equals the reference's writer byte for
    byte: awkward magnitudes, subnormals, -0, integers beyond 2^24 (printed
    exactly), and a smoothed volume's real curve."""
    import torch
    if not oracle.ref_available():
        pytest.skip("reference not compiled here")
    rng = np.random.default_rng(11)
    t = np.concatenate([
        rng.random(500).astype(np.float32) * np.float32(10.0) ** rng.integers(-40, 38, 500).astype(np.float32),
        np.array([0.0, -0.0, 1e-45, 1.17549435e-38, 1.5258789e-05, 0.0001, 0.001, 123456.0, 1e7,
                  16777216.0, 50331648.0, 1.2e6, 3.4028235e38, -2.5], np.float32)])
    t = t[np.isfinite(t)]
    chi = rng.integers(-2 ** 40, 2 ** 40, t.size)
    got = ctx.format_curve(t, chi, fmt)
    if fmt == "csv":
        assert got == oracle.ref_csv(t, chi)
    else:
        assert got == _ref_writer_py(t, chi, fmt)
    # the device-array path and a real curve of a smoothed field
    x = torch.empty((24, 30, 36), dtype=torch.float32, device="cuda")
    ctx.uniform_noise(x, seed=4)
    y = ctx.gaussian_smooth(x, 1.5, 5)
    cur = ctx.curve(y.cpu().numpy())
    dev_t = torch.from_numpy(np.ascontiguousarray(cur.thresholds)).cuda()
    dev_c = torch.from_numpy(np.ascontiguousarray(cur.chi)).cuda()
    got = ctx.format_curve(dev_t, dev_c, fmt)
    if fmt == "csv":
        assert got == oracle.ref_csv(cur.thresholds, cur.chi)
    else:
        assert got == _ref_writer_py(cur.thresholds, cur.chi, fmt)


def test_format_curve_integer_thresholds(ctx):
    img = oracle.synth("u8", (64, 64), seed=2)
    cur = ctx.curve(img)
    assert ctx.format_curve(cur.thresholds, cur.chi, "csv") == oracle.ref_csv(cur.thresholds, cur.chi)
    t16 = np.array([0, 7, 65535], np.uint16)
    assert ctx.format_curve(t16, np.array([1, -2, 3]), "json") == b'[{"t":0,"chi":1},{"t":7,"chi":-2},{"t":65535,"chi":3}]\n'
    assert ctx.format_curve(np.zeros(0, np.float32), np.zeros(0, np.int64), "json") == b"[]\n"
