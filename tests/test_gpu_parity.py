"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
golden fixtures.  Bit-exact everywhere -- this is integer work."""
import numpy as np
import pytest

import oracle
import paper_2203_09087_b200 as eb

pytestmark = pytest.mark.gpu


def _img(rec):
    return np.array(rec["image"], dtype=rec["dtype"]).reshape(rec["shape"])


def _same(a_vals, a_ch, b_vals, b_ch):
    a_vals, b_vals = np.asarray(a_vals), np.asarray(b_vals)
    if a_vals.dtype == np.float32 or b_vals.dtype == np.float32:
        ok_v = np.array_equal(np.asarray(a_vals, np.float32).view(np.uint32),
                              np.asarray(b_vals, np.float32).view(np.uint32))
    else:
        ok_v = np.array_equal(a_vals.astype(np.int64), b_vals.astype(np.int64))
    return ok_v and np.array_equal(np.asarray(a_ch, np.int64), np.asarray(b_ch, np.int64))


def test_hand_fixtures(ctx, golden):
    for name, rec in golden["hand"].items():
        img = _img(rec)
        got = ctx.vcec(img)
        assert _same(got.values, got.changes, np.array(rec["values"], img.dtype), rec["changes"]), name


def test_random_fixtures(ctx, golden):
    for rec in golden["random"]:
        img = _img(rec)
        got = ctx.vcec(img)
        assert _same(got.values, got.changes, np.array(rec["values"], img.dtype), rec["changes"])


def _random_images(seed, n, maxd2=9, maxd3=7):
    rng = np.random.default_rng(seed)
    for t in range(n):
        d = (int(rng.integers(1, maxd2)), int(rng.integers(1, maxd2))) if t % 2 == 0 else \
            tuple(int(x) for x in rng.integers(1, maxd3, 3))
        k = t % 3
        if k == 0:
            yield rng.integers(0, 8, d).astype(np.uint8)
        elif k == 1:
            yield rng.random(5).astype(np.float32)[rng.integers(0, 5, d)]
        else:
            yield rng.integers(0, 6, d).astype(np.uint16)


def test_oracle_sweep_whole_volume(ctx):
    # acceptance.cpp:95-142 shapes, resident volume path
    for img in _random_images(1, 300):
        a = ctx.vcec(img)
        b = oracle.vcec(img)
        assert _same(a.values, a.changes, *b), (img.shape, img.dtype)


def test_oracle_sweep_chunked_stream(ctx):
    # chunk invariance through the streaming driver (chunks {1,2,3,w0})
    for img in _random_images(2, 120):
        b = oracle.vcec(img)
        w0 = img.shape[0]
        for c in sorted({1, 2, 3, w0}):
            plan = eb.plan_chunks(eb.Dims.of(img.shape), eb.ChunkTarget.count(c))
            a = eb.process_image(img, plan)
            assert _same(a.values, a.changes, *b), (img.shape, c)


def test_medium_shapes_u8(ctx):
    rng = np.random.default_rng(3)
    for shape in [(37, 41, 29), (64, 64, 64), (5, 300, 7), (130, 1, 70), (1, 1, 1000), (257, 255, 1),
                  (64, 1024, 1), (3, 3, 513)]:
        img = rng.integers(0, 256, shape).astype(np.uint8)
        a = ctx.vcec(img)
        assert _same(a.values, a.changes, *oracle.vcec(img)), shape


def test_medium_shapes_u16_and_smooth(ctx):
    rng = np.random.default_rng(4)
    for shape in [(33, 47, 51), (200, 300, 1), (16, 16, 16)]:
        img = rng.integers(0, 65536, shape).astype(np.uint16)
        a = ctx.vcec(img)
        assert _same(a.values, a.changes, *oracle.vcec(img)), shape
    # plateau field ((x>>3)+(y>>3)+(z>>3)) & 255 (SURVEY.md 8(d) robustness)
    z, y, x = np.meshgrid(np.arange(40), np.arange(48), np.arange(56), indexing="ij")
    img = (((x >> 3) + (y >> 3) + (z >> 3)) & 255).astype(np.uint8)
    a = ctx.vcec(img)
    assert _same(a.values, a.changes, *oracle.vcec(img))
    const = np.full((20, 30, 40), 7, np.uint8)
    a = ctx.vcec(const)
    assert list(a.values) == [7] and list(a.changes) == [1]


def test_f32_sorted_and_affine(ctx):
    rng = np.random.default_rng(5)
    img = rng.random((24, 31, 17)).astype(np.float32)
    img[0, 0, 0] = -0.0
    img[3, 4, 5] = 0.0
    img[5, 5, 5] = np.inf
    img[23, 30, 16] = -np.inf
    a = ctx.vcec(img)  # general path: device sort + reduce-by-key
    assert _same(a.values, a.changes, *oracle.vcec(img))
    q = (rng.integers(0, 65536, (40, 33, 29)) * 2.0 ** -16).astype(np.float32)
    a = ctx.vcec(q, binmap=eb.quantised_binmap(65536))
    assert _same(a.values, a.changes, *oracle.vcec(q))
    bad = q.copy()
    bad[1, 1, 1] = 0.3  # not on the 2^-16 grid
    with pytest.raises(eb.EccError) as ei:
        ctx.vcec(bad, binmap=eb.quantised_binmap(65536))
    assert ei.value.code == eb.ECC_EBINMAP
    nan = q.copy()
    nan[2, 2, 2] = np.nan
    with pytest.raises(eb.EccError):
        ctx.vcec(nan)


def test_config1_golden(ctx, golden):
    img = oracle.synth("u8", (256, 256))
    c = ctx.curve(img)
    assert oracle.curve_digest(c.thresholds, c.chi) == golden["configs"]["C1"]["digest"]


@pytest.mark.slow
def test_config2_golden_device_resident(ctx, golden):
    import torch
    vol = torch.empty((512, 512, 512), dtype=torch.uint8, device="cuda")
    ctx.fill_synthetic(vol, seed=1)
    torch.cuda.synchronize()
    c = ctx.curve(vol)
    g = golden["configs"]["C2"]
    assert oracle.curve_digest(c.thresholds, c.chi) == g["digest"]
    # the device generator agrees with the oracle's host generator
    host = oracle.synth("u8", (512, 512, 512))
    assert np.array_equal(vol.cpu().numpy(), host)


@pytest.mark.slow
def test_config3_images_golden(ctx, golden):
    for b in (0, 4095):
        img = oracle.synth("u16", (512, 512), seed=1, base=b * 512 * 512)
        c = ctx.curve(img)
        assert oracle.curve_digest(c.thresholds, c.chi) == golden["configs"][f"C3_{b}"]["digest"]
        chi, pres = ctx.batch2d(img[None])
        t, cc = eb.curve_batch_to_points(chi[0], pres[0])
        assert oracle.curve_digest(t, cc) == golden["configs"][f"C3_{b}"]["digest"]


def test_batch2d_small(ctx):
    rng = np.random.default_rng(6)
    for dt, hi in ((np.uint8, 256), (np.uint16, 65536), (np.uint8, 4), (np.uint16, 3)):
        imgs = rng.integers(0, hi, (9, 37, 23)).astype(dt)
        chi, pres = ctx.batch2d(imgs)
        for b in range(imgs.shape[0]):
            t, cc = eb.curve_batch_to_points(chi[b], pres[b])
            v, c = oracle.curve(imgs[b])
            assert np.array_equal(t, v.astype(np.int64)) and np.array_equal(cc, c)


def test_batch2d_constant_images_spill(ctx):
    # one bin receives every pixel: exercises the packed-bin overflow spill
    imgs = np.zeros((2, 512, 512), np.uint16)
    imgs[1] = 40000
    imgs[1, ::2, ::2] = 7  # isolated minima -> large positive partial sums
    chi, pres = ctx.batch2d(imgs)
    for b in range(2):
        t, cc = eb.curve_batch_to_points(chi[b], pres[b])
        v, c = oracle.curve(imgs[b])
        assert np.array_equal(t, v.astype(np.int64)) and np.array_equal(cc, c)


def test_slabs_sum_to_whole(ctx):
    import torch
    rng = np.random.default_rng(8)
    img = rng.integers(0, 256, (50, 40, 30)).astype(np.uint8)
    whole = torch.zeros(512, dtype=torch.int64, device="cuda")
    dev = torch.from_numpy(img).cuda()
    ctx.accumulate_slab(dev, eb.Dims.of(img.shape), 0, 0, 50, whole)
    parts = torch.zeros(512, dtype=torch.int64, device="cuda")
    for a, b in ((0, 13), (13, 14), (14, 37), (37, 50)):
        p0 = max(a - 1, 0)
        p1 = min(b + 1, 50)
        ctx.accumulate_slab(dev[p0:p1].contiguous(), eb.Dims.of(img.shape), p0, a, b, parts)
    torch.cuda.synchronize()
    assert torch.equal(whole, parts)
    h, cnt = oracle.hist_dense(img)
    assert np.array_equal(whole[:256].cpu().numpy(), h)
    assert np.array_equal(whole[256:].cpu().numpy(), cnt)


def test_compute_changes_matches_oracle(ctx):
    import torch
    rng = np.random.default_rng(9)
    # (24, 40, 48) / (17, 35, 64) / (40, 70, 96): rows a multiple of 16 bytes -> the TMA-fed
    # bit-sliced kernel's changes mode; (20, 21, 22) -> the tournament kernel; (30, 40, 1) 2D
    for shape, hi in [((20, 21, 22), 5), ((30, 40, 1), 5), ((24, 40, 48), 5), ((17, 35, 64), 256),
                      ((40, 70, 96), 3)]:
        img = rng.integers(0, hi, shape).astype(np.uint8)
        dev = torch.from_numpy(img).cuda()
        out = torch.full((img.size,), 99, dtype=torch.int8, device="cuda")
        ctx.compute_changes(dev, eb.Dims.of(shape), 0, 0, shape[0], out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(shape), oracle.changes(img)), shape
    # a slab of the TMA-shaped volume: owned planes [5, 19) with their halo planes only
    shape = (24, 40, 48)
    img = rng.integers(0, 7, shape).astype(np.uint8)
    want = oracle.changes(img)[5:19]
    slab = torch.from_numpy(np.ascontiguousarray(img[4:20])).cuda()
    out = torch.full((14 * 40 * 48,), 99, dtype=torch.int8, device="cuda")
    ctx.compute_changes(slab, eb.Dims.of(shape), 4, 5, 19, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().reshape(want.shape), want)


def test_stream_failure_names_chunk(ctx):
    # test_streaming.cpp:164-198 (FlakySource)
    rng = np.random.default_rng(53)
    img = rng.random((8, 3, 3)).astype(np.float32)

    class Flaky(eb.MemorySource):
        def read_rows(self, r0, r1, dst):
            if r1 > 5:
                raise RuntimeError("simulated device failure")
            super().read_rows(r0, r1, dst)

    plan = eb.plan_chunks(eb.Dims.of(img.shape), eb.ChunkTarget.count(4))
    with pytest.raises(eb.EccError) as ei:
        eb.process_image(Flaky(img), plan)
    assert "chunk" in str(ei.value) and "simulated device failure" in str(ei.value)


def test_invalid_plans_rejected(ctx):
    img = np.array([[1], [2], [3], [4]], np.float32).reshape(4, 1, 1)
    src = eb.MemorySource(img)
    for ranges in ([], [(0, 2), (3, 4)], [(0, 2), (2, 3)], [(1, 4)]):
        plan = eb.ChunkPlan([eb.ChunkRange(a, b) for a, b in ranges])
        with pytest.raises(eb.EccError):
            ctx.process_source(src, plan)


def test_stream_reports_timings_and_overlap(ctx):
    rng = np.random.default_rng(59)
    img = rng.integers(0, 256, (160, 128, 128)).astype(np.uint8)
    plan = eb.plan_chunks(eb.Dims.of(img.shape), eb.ChunkTarget.count(4))
    rep = eb.EngineReport()
    v = eb.process_image(img, plan, eb.EngineOptions(ingest_delay_ms=50), rep)
    assert v.total() == 1
    assert len(rep.chunks) == 4
    for t in rep.chunks:
        assert t.ingest_end >= t.ingest_begin and t.kernel_end >= t.kernel_begin
    # acceptance.cpp:293-317: ingest of chunk k+1 overlaps device work of chunk k
    assert any(min(rep.chunks[k].kernel_end, rep.chunks[k + 1].ingest_end) >
               max(rep.chunks[k].kernel_begin, rep.chunks[k + 1].ingest_begin) or
               rep.chunks[k + 1].ingest_begin < rep.chunks[k].kernel_end
               for k in range(3))


def test_process_host_direct_dma(ctx):
    """ecc_process_host: chunks + halos DMA'd straight from a (pinned) host
    buffer, three device slabs in flight; every type it supports, several
    plans, against the oracle."""
    import torch
    rng = np.random.default_rng(77)
    cases = [rng.integers(0, 256, (37, 40, 48)).astype(np.uint8),        # fast u8 path
             rng.integers(0, 256, (23, 17, 19)).astype(np.uint8),        # generic u8
             rng.integers(0, 3000, (15, 21, 9)).astype(np.uint16),
             rng.integers(0, 256, (30, 40, 1)).astype(np.uint8)]         # 2D
    for img in cases:
        want = oracle.vcec(img)
        pinned = torch.from_numpy(img).pin_memory().numpy()
        for c in (1, 2, 5, img.shape[0]):
            plan = eb.plan_chunks(eb.Dims.of(img.shape), eb.ChunkTarget.count(c))
            rep = eb.EngineReport()
            got = ctx.process_host(pinned, plan, report=rep)
            assert _same(got.values, got.changes, *want), (img.shape, c)
            assert len(rep.chunks) == len(plan.ranges)
    q = (rng.integers(0, 65536, (12, 10, 14)) * 2.0 ** -16).astype(np.float32)
    got = ctx.process_host(q, eb.plan_chunks(eb.Dims.of(q.shape), eb.ChunkTarget.count(3)),
                           binmap=eb.quantised_binmap(65536))
    assert _same(got.values, got.changes, *oracle.vcec(q))


@pytest.mark.slow
def test_config5_first_64_planes_streamed(ctx, golden):
    import torch
    side = 4096
    host = torch.empty((64, side, side), dtype=torch.uint8, pin_memory=True)
    dev = torch.empty((64, side, side), dtype=torch.uint8, device="cuda")
    ctx.fill_synthetic(dev, seed=1)
    host.copy_(dev)
    del dev
    v = ctx.process_host(host.numpy(), eb.plan_chunks(eb.Dims(64, side, side), eb.ChunkTarget.count(8)))
    cur = eb.vcec_to_ecc(v)
    assert oracle.curve_digest(cur.thresholds, cur.chi) == golden["configs"]["C5_64"]["digest"]


@pytest.mark.slow
def test_config4_golden_device_resident(ctx, golden):
    import torch
    vol = torch.empty((1024, 1024, 1024), dtype=torch.float32, device="cuda")
    ctx.fill_synthetic(vol, seed=1)
    c = ctx.curve(vol, binmap=eb.quantised_binmap(65536))
    assert oracle.curve_digest(c.thresholds, c.chi) == golden["configs"]["C4"]["digest"]
    assert c.size() == 65536 and int(c.chi[-1]) == 1


def test_process_file_raw_and_big_endian(ctx, tmp_path):
    """FileSource semantics (chunk.hpp:154-189, image.hpp:39-52) with the f32
    byte swap and NaN check on the GPU; error wording as the reference."""
    rng = np.random.default_rng(12)
    img = rng.random((9, 7, 5)).astype(np.float32)
    img[3, 2, 1] = -0.0
    dims = eb.Dims.of(img.shape)
    plan = eb.plan_chunks(dims, eb.ChunkTarget.count(3))
    want = oracle.vcec(img)
    le, be = tmp_path / "le.raw", tmp_path / "be.raw"
    img.tofile(le)
    img.astype(">f4").tofile(be)
    for path, big in ((le, False), (be, True)):
        got = ctx.process_file(str(path), dims, np.float32, plan, big_endian=big)
        assert _same(got.values, got.changes, *want), path
    u8 = rng.integers(0, 256, (12, 16, 32)).astype(np.uint8)
    p8 = tmp_path / "u8.raw"
    u8.tofile(p8)
    got = ctx.process_file(str(p8), eb.Dims.of(u8.shape), np.uint8,
                           eb.plan_chunks(eb.Dims.of(u8.shape), eb.ChunkTarget.count(4)))
    assert _same(got.values, got.changes, *oracle.vcec(u8))
    # NaN: first chunk (in plan order) whose rows hold one, reference wording
    bad = img.copy()
    bad[5, 1, 2] = np.nan
    pb = tmp_path / "nan.raw"
    bad.tofile(pb)
    with pytest.raises(eb.EccError) as ei:
        ctx.process_file(str(pb), dims, np.float32, plan)
    idx = (5 * 7 + 1) * 5 + 2
    assert f"NaN value at linear index {idx}" in str(ei.value) and "chunk" in str(ei.value)
    with pytest.raises(eb.EccError) as ei:
        ctx.process_file(str(le), eb.Dims(9, 7, 4), np.float32)
    assert "size mismatch" in str(ei.value)
    with pytest.raises(eb.EccError) as ei:
        ctx.process_file(str(tmp_path / "missing.raw"), dims, np.float32)
    assert "cannot open" in str(ei.value)


def test_acceptance_sweep_1000_images(ctx):
    """acceptance.cpp:95-142: 1000 random images (dims {1..8}^2 and {1..6}^3,
    u8 values 0..7, f32 drawn from a pool of 5 values), every chunking in
    {1, 2, 3, w0}, equal to the oracle."""
    rng = np.random.default_rng(2024)
    pool = np.array([-1.5, 0.0, 0.25, 3.0, 7.5], np.float32)
    for t in range(1000):
        d = (tuple(int(x) for x in rng.integers(1, 9, 2)) if t % 2 == 0 else
             tuple(int(x) for x in rng.integers(1, 7, 3)))
        img = (rng.integers(0, 8, d).astype(np.uint8) if t % 4 < 2 else
               pool[rng.integers(0, 5, d)])
        want = oracle.vcec(img)
        cs = {1, 2, 3, img.shape[0]} if t % 10 == 0 else {1 + t % 3}
        for c in sorted(cs):
            plan = eb.plan_chunks(eb.Dims.of(img.shape), eb.ChunkTarget.count(c))
            got = eb.process_image(img, plan)
            assert _same(got.values, got.changes, *want), (t, img.shape, c)


def test_order_only_dependence(ctx):
    """test_kernel.cpp:175-200: only the order of values matters -- a strictly
    increasing remap leaves every change unchanged."""
    rng = np.random.default_rng(31)
    for shape in [(20, 30, 40), (64, 64, 1), (9, 16, 48)]:
        img = rng.integers(0, 256, shape).astype(np.uint8)
        a = ctx.vcec(img)
        f = (img.astype(np.float32) * 0.5 - 3.0).astype(np.float32)
        b = ctx.vcec(f)
        u = (img.astype(np.uint16) * 200 + 7).astype(np.uint16)
        c = ctx.vcec(u)
        assert np.array_equal(a.changes, b.changes) and np.array_equal(a.changes, c.changes)


def test_chunk_invariance_64_cubed_bitwise(ctx):
    """acceptance.cpp:203-227: bitwise-identical curves over chunk counts
    1..8 on 64^3 (u8 through the fast path, f32 through the sorted path)."""
    rng = np.random.default_rng(64)
    u8 = rng.integers(0, 256, (64, 64, 64)).astype(np.uint8)
    f32 = rng.integers(0, 40, (64, 64, 64)).astype(np.float32) * np.float32(0.125)
    for img in (u8, f32):
        ref = None
        for c in range(1, 9):
            plan = eb.plan_chunks(eb.Dims.of(img.shape), eb.ChunkTarget.count(c))
            v = eb.process_image(img, plan)
            cur = eb.vcec_to_ecc(v)
            key = (cur.thresholds.tobytes(), cur.chi.tobytes())
            ref = ref or key
            assert key == ref, c
        assert np.array_equal(v.changes, oracle.vcec(img)[1])


def test_memory_budget_plan_streams_out_of_core_shape(ctx):
    """acceptance.cpp:253-290: a 1024 x 256^2 f32 volume planned under a
    64 MiB budget streams chunk by chunk and matches the whole-volume result."""
    rng = np.random.default_rng(5)
    img = (rng.integers(0, 1000, (1024, 256, 256)).astype(np.float32) * np.float32(0.001))
    dims = eb.Dims.of(img.shape)
    plan = eb.plan_chunks(dims, eb.ChunkTarget.memory_budget(64 << 20), dtype=np.float32)
    assert plan.chunk_count() > 8
    for r in plan.ranges:
        assert eb.padded_chunk_bytes(dims, r.len(), np.float32) <= 64 << 20
    v = eb.process_image(img, plan)
    assert v.total() == 1
    q = ctx.vcec(img)
    assert np.array_equal(v.changes, q.changes)


@pytest.mark.slow
def test_u16_spill_path_isolated_minima(ctx):
    """Adversarial input for the packed 16-bit shared histogram of the u16
    kernel: 256^3 isolated minima share one value, so that bin's running
    sum crosses the +-16384 band many times in every CTA and the exact spill
    path runs; the whole VCEC must still equal the oracle's."""
    rng = np.random.default_rng(99)
    img = rng.integers(1000, 60000, (512, 512, 512)).astype(np.uint16)
    img[::2, ::2, ::2] = 0
    got = ctx.vcec(img)
    v, c = oracle.vcec(img)
    assert np.array_equal(got.values.astype(np.int64), v.astype(np.int64))
    assert np.array_equal(got.changes, c)
    assert got.changes[0] == 256 ** 3


def _minus7_lattice(shape, a, b, c):
    """2 x 2 x 2-periodic lattice whose class-(even, even, even) voxels all
    have change -7 (the most negative 3D change): value `a`
    there, `c` < a on the (odd, odd, odd) corners, `b` > a elsewhere -- each
    such voxel wins its 6 face pairs and 12 edge quads and no cube, -1 + 6 -
    12 + 0 = -7 -- so one bin takes -7 from an eighth of all voxels."""
    x, y, z = np.indices(shape)
    img = np.full(shape, b, dtype=np.uint16)
    img[(x % 2 == 0) & (y % 2 == 0) & (z % 2 == 0)] = a
    img[(x % 2 == 1) & (y % 2 == 1) & (z % 2 == 1)] = c
    return img


@pytest.mark.parametrize("shape", [(64, 96, 256), (130, 66, 300)])
def test_hist16_adversarial_minus7_lattice(ctx, shape):
    """The packed 16-bit histogram's worst case (hist16.cuh bound): every
    value-`a` voxel pushes the same half down by 7, so every CTA's half
    crosses the band again and again and the exact compare-and-swap spill
    runs under full contention; the VCEC must equal the oracle's."""
    img = _minus7_lattice(shape, 1000, 50000, 7)
    got = ctx.vcec(img)
    v, c = oracle.vcec(img)
    assert _same(got.values, got.changes, v, c)
    n_a = int(((np.indices(shape) % 2) == 0).all(axis=0).sum())
    i = int(np.searchsorted(v, 1000))
    assert c[i] <= -7 * n_a // 2  # the adversarial bin really is hot
    # the same lattice as quantised f32 through the affine key pass
    f = img.astype(np.float32) * np.float32(2.0 ** -16)
    got = ctx.vcec(f, binmap=eb.quantised_binmap(65536))
    assert np.array_equal(got.changes, c)


def test_f32_sorted_2d_infinities_and_signed_zeros(ctx):
    """The reference's quirks on the sorted f32 path in 2D:
    +inf pixels tie with the +inf collar sentinel, -0 merges into +0."""
    rng = np.random.default_rng(77)
    for shape in [(30, 41), (1, 50), (64, 1)]:
        img = rng.choice(np.array([-np.inf, -1.5, -0.0, 0.0, 2.0, np.inf], np.float32),
                         size=shape)
        a = ctx.vcec(img)
        assert _same(a.values, a.changes, *oracle.vcec(img)), shape
        if oracle.ref_available():
            assert _same(a.values, a.changes, *oracle.ref_vcec(img)), shape


def test_randomised_differential_smoke():
    """tools/fuzz.py for 15 s: random dtype / shape / value range / public
    path against the oracle (a 240 s run: profiles/r01m_fuzz.json)."""
    import subprocess
    import sys as _sys
    import os as _os
    root = _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))
    r = subprocess.run([_sys.executable, _os.path.join(root, "tools", "fuzz.py"), "15", "7"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and " 0 failures" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("lo,hi", [(0, 2), (7, 9), (65530, 65536), (1000, 1006)])
@pytest.mark.parametrize("shape", [(2000, 512), (2000, 1024), (2035, 1197), (1200, 300)])
def test_hot_bins_packed_histogram(ctx, lo, hi, shape):
    """Images with only a few distinct values: one CTA accumulates per-bin
    sums far beyond the 16-bit halves of the packed 65536-bin table (both
    batched kernels); the exact compare-and-swap spill keeps them exact."""
    rng = np.random.default_rng(lo + shape[1])
    img = rng.integers(lo, hi, shape).astype(np.uint16)
    chi, pres = ctx.batch2d(img[None])
    t, cc = eb.curve_batch_to_points(chi[0], pres[0].view(np.uint32))
    v, c = oracle.vcec(img)
    assert np.array_equal(t, v.astype(np.int64)) and np.array_equal(cc, np.cumsum(c))
    a = ctx.vcec(img)
    assert np.array_equal(a.changes, c)


@pytest.mark.parametrize("shape", [(2000, 32, 40), (400, 64, 64), (200000, 32), (3000, 2000)])
def test_hot_bins_16bit_kernels(ctx, shape):
    """Two-valued u16 / quantised-f32 images through the 3D and single-image
    2D 16-bit kernels (each CTA sees bins with sums far beyond 16 bits)."""
    rng = np.random.default_rng(len(shape) + shape[0])
    img = rng.integers(5, 7, shape).astype(np.uint16)
    a = ctx.vcec(img)
    v, c = oracle.vcec(img)
    assert np.array_equal(a.values.astype(np.int64), v.astype(np.int64))
    assert np.array_equal(a.changes, c)
    q = (img.astype(np.float64) * 2.0 ** -16).astype(np.float32)
    b = ctx.vcec(q, binmap=eb.quantised_binmap(65536))
    assert np.array_equal(b.changes, c)


@pytest.mark.parametrize("case", ["smoothed", "narrow", "wide", "few", "signed_zero_inf"])
def test_f32_sorted_dense_and_sort_paths(ctx, case):
    """General f32 volumes of >= 2^20 voxels: order-key spans < 2^24 take the
    dense key histogram (no sort), wider spans the radix sort; both equal the
    oracle's (value, summed change) list."""
    rng = np.random.default_rng(hash(case) % 1000)
    shape = (64, 128, 160)
    if case == "smoothed":
        img = oracle.gaussian_smooth(oracle.uniform_noise(shape, 3), 2.0, 13)
    elif case == "narrow":
        img = (0.75 + rng.random(shape) * 2.0 ** -8).astype(np.float32)
    elif case == "wide":
        img = (rng.standard_normal(shape) * 1e3).astype(np.float32)
    elif case == "few":
        img = rng.choice(np.array([0.1, 0.2, 0.3], np.float32), size=shape)
    else:
        img = rng.choice(np.array([-0.0, 0.0, 1.0, np.inf], np.float32), size=shape)
    a = ctx.vcec(img)
    v, c = oracle.vcec(img)
    assert np.array_equal(np.asarray(a.values, np.float32).view(np.uint32), np.asarray(v, np.float32).view(np.uint32))
    assert np.array_equal(a.changes, c)
    import torch
    b = ctx.vcec(torch.from_numpy(img).cuda())
    assert np.array_equal(b.changes, c)


def test_f32_sorted_dense_streamed_slabs(ctx):
    """Streamed general f32 (>= 2^20 voxels per slab): every slab takes the
    dense key histogram with its own key range, the runs merge on the device."""
    rng = np.random.default_rng(8)
    img = (2.0 + rng.random((96, 128, 256)) * 2.0 ** -7).astype(np.float32)
    img[:, :, ::7] = np.round(img[:, :, ::7] * 256) / 256  # ties across slabs
    v, c = oracle.vcec(img)
    for chunks in (1, 2, 3):
        plan = eb.plan_chunks(eb.Dims.of(img.shape), eb.ChunkTarget.count(chunks))
        got = eb.process_image(img, plan)
        assert np.array_equal(np.asarray(got.values, np.float32).view(np.uint32),
                              np.asarray(v, np.float32).view(np.uint32)), chunks
        assert np.array_equal(got.changes, c), chunks


@pytest.mark.parametrize("case", ["u16", "u16_odd", "f32_affine"])
def test_overlapped_host_input_dense_maps(ctx, case):
    """Large host volumes with the other dense maps take the overlapped path
    (chunked H2D, per-chunk K1+K2 on slab views, K3 after the last)."""
    rng = np.random.default_rng(len(case))
    if case == "u16":
        img, bm = rng.integers(0, 65536, (128, 512, 256)).astype(np.uint16), None
    elif case == "u16_odd":
        img, bm = rng.integers(0, 300, (100, 400, 420)).astype(np.uint16), None
    else:
        img = (rng.integers(0, 65536, (64, 512, 256)) * 2.0 ** -16).astype(np.float32)
        bm = eb.quantised_binmap(65536)
    a = ctx.vcec(img, binmap=bm) if bm else ctx.vcec(img)
    v, c = oracle.vcec(img)
    assert np.array_equal(a.changes, c)
    if img.dtype == np.float32:
        assert np.array_equal(np.asarray(a.values, np.float32).view(np.uint32), v.astype(np.float32).view(np.uint32))
    else:
        assert np.array_equal(a.values.astype(np.int64), v.astype(np.int64))
    if case == "f32_affine":
        bad = img.copy()
        bad[40, 7, 9] = 0.3
        with pytest.raises(eb.EccError):
            ctx.vcec(bad, binmap=bm)


def test_f32_more_distinct_values_than_the_first_capacity(ctx):
    """The Python wrapper first asks for 4 M points; a volume with more
    distinct f32 values (almost one per voxel here) gets the exact count back
    and is called again at that size (ecc_vcec reports the count with the
    capacity error).  Both the VCEC and the curve stay bit-exact."""
    rng = np.random.default_rng(41)
    img = rng.standard_normal((264, 128, 128), dtype=np.float32)  # ~all distinct
    got = ctx.vcec(img)
    v, c = oracle.vcec(img)
    assert got.size() > (1 << 22)
    assert np.array_equal(np.asarray(got.values), v) and np.array_equal(np.asarray(got.changes), c)
    cur = ctx.curve(img)
    assert np.array_equal(np.asarray(cur.chi), np.cumsum(c))


@pytest.mark.parametrize("count,h,w", [(9, 37, 32), (3, 1, 16), (5, 300, 48), (2, 64, 512),
                                       (1, 700, 1024), (4, 33, 2000), (300, 17, 64),
                                       (2, 1000, 96)])
def test_batch2d_u8_bit_sliced(ctx, count, h, w):
    """u8 batches whose rows are a multiple of 16 bytes run the bit-sliced
    k_u8_2d kernel, one thread-block cluster per image (several CTAs per
    image when the batch is small; rows packed or in strips by width); the
    dense chi rows and occupancy bitmaps match the oracle image by image --
    random values, ties at the collar value 255, and the dense row format
    (every value 0..255, absent ones carrying the running sum)."""
    import torch
    rng = np.random.default_rng(count * 1000 + w)
    imgs = rng.integers(0, 256, (count, h, w)).astype(np.uint8)
    imgs[:, :, ::5] = 255
    imgs[count // 2] = rng.integers(0, 3, (h, w))  # few values: long runs of absent ones
    for src in (imgs, torch.from_numpy(imgs).cuda()):
        chi, pres = ctx.batch2d(src)
        if not isinstance(chi, np.ndarray):
            torch.cuda.synchronize()
            chi, pres = chi.cpu().numpy(), pres.cpu().numpy().view(np.uint32)
        for b in range(count):
            v, c = oracle.vcec(imgs[b])
            dense = np.zeros(256, np.int64)
            dense[v.astype(np.int64)] = c
            assert np.array_equal(chi[b].astype(np.int64), np.cumsum(dense)), (b, h, w)
            bits = np.unpackbits(pres[b].astype("<u4").view(np.uint8), bitorder="little")[:256]
            assert np.array_equal(np.nonzero(bits)[0], v.astype(np.int64)), (b, h, w)


def test_batch2d_u8_more_images_than_grid_y(ctx):
    """More than 65535 images (the grid's y limit): the bit-sliced batch is
    launched in slices; images on both sides of the cut are exact."""
    import torch
    rng = np.random.default_rng(3)
    imgs = rng.integers(0, 256, (70001, 3, 16)).astype(np.uint8)
    chi, pres = ctx.batch2d(torch.from_numpy(imgs).cuda())
    torch.cuda.synchronize()
    chi, pres = chi.cpu().numpy(), pres.cpu().numpy().view(np.uint32)
    for b in (0, 1, 65534, 65535, 65536, 70000):
        t, cc = eb.curve_batch_to_points(chi[b], pres[b])
        v, c = oracle.curve(imgs[b])
        assert np.array_equal(t, v.astype(np.int64)) and np.array_equal(cc, c), b
