"""Small invocations of every device path, for compute-sanitizer
(memcheck / racecheck / synccheck).  Each result is checked against the
oracle so a sanitizer run is also a parity run.

  compute-sanitizer --tool memcheck python tools/sanitize_driver.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2203_09087_b200 as eb  # noqa: E402

ctx = eb.context(0)
rng = np.random.default_rng(0)
ok = True


def check(name, got, img):
    global ok
    v, c = oracle.vcec(img)
    good = np.array_equal(np.asarray(got.changes), c)
    ok &= good
    print(("ok  " if good else "BAD ") + name, flush=True)


for shape in [(9, 33, 48), (5, 7, 20), (64, 1, 100)]:
    img = rng.integers(0, 256, shape).astype(np.uint8)
    check(f"u8 3D {shape}", ctx.vcec(img), img)
for shape in [(40, 1000), (3, 5), (17, 961)]:
    img = rng.integers(0, 256, shape).astype(np.uint8)
    check(f"u8 2D {shape}", ctx.vcec(img), img)
    img16 = rng.integers(0, 65536, shape).astype(np.uint16)
    check(f"u16 2D {shape}", ctx.vcec(img16), img16)
img16 = rng.integers(0, 65536, (12, 40, 48)).astype(np.uint16)
check("u16 3D", ctx.vcec(img16), img16)
# column-layout boundaries (first / last columns with a virtual collar, bits.cuh cols)
for shape in [(4, 62, 64), (3, 93, 96), (2, 512, 512), (3, 32, 32)]:
    img = rng.integers(250, 256, shape).astype(np.uint8)
    check(f"u8 3D columns {shape}", ctx.vcec(img), img)
for shape in [(4, 62, 64), (3, 93, 40), (2, 512, 512)]:
    img16 = rng.integers(0, 65536, shape).astype(np.uint16)
    check(f"u16 3D columns {shape}", ctx.vcec(img16), img16)
q = (rng.integers(0, 65536, (10, 33, 40)) * 2.0 ** -16).astype(np.float32)
check("f32 affine 3D", ctx.vcec(q, binmap=eb.quantised_binmap(65536)), q)
q2 = (rng.integers(0, 65536, (50, 70)) * 2.0 ** -16).astype(np.float32)
check("f32 affine 2D", ctx.vcec(q2, binmap=eb.quantised_binmap(65536)), q2)
f = rng.random((11, 13, 17)).astype(np.float32)
check("f32 sorted 3D", ctx.vcec(f), f)
f2 = rng.random((30, 40)).astype(np.float32)
check("f32 sorted 2D", ctx.vcec(f2), f2)
for dt, hi in ((np.uint8, 256), (np.uint16, 65536)):
    img = rng.integers(0, hi, (40, 24, 36)).astype(dt)
    plan = eb.plan_chunks(eb.Dims.of(img.shape), eb.ChunkTarget.count(3), dt)
    check(f"process_host {dt.__name__}", eb.process_image(img, plan), img)
    opts = eb.EngineOptions(ingest_delay_ms=0.1)
    check(f"process_stream {dt.__name__}", eb.process_image(img, plan, opts), img)
imgs = rng.integers(0, 65536, (3, 31, 45)).astype(np.uint16)
chi, pres = ctx.batch2d(imgs)
for b in range(3):
    t, cc = eb.curve_batch_to_points(chi[b], pres[b])
    v, c = oracle.vcec(imgs[b])
    good = np.array_equal(t, v.astype(np.int64)) and np.array_equal(cc, np.cumsum(c))
    ok &= good
    print(("ok  " if good else "BAD ") + f"batch2d u16 #{b}", flush=True)
imgsv = rng.integers(0, 65536, (2, 64, 512)).astype(np.uint16)  # C3-shaped rows: cp.async staging
chi, pres = ctx.batch2d(imgsv)
for b in range(2):
    t, cc = eb.curve_batch_to_points(chi[b], pres[b])
    v, c = oracle.vcec(imgsv[b])
    good = np.array_equal(t, v.astype(np.int64)) and np.array_equal(cc, np.cumsum(c))
    ok &= good
    print(("ok  " if good else "BAD ") + f"batch2d u16 512-wide #{b}", flush=True)
# general f32 over >= 2^20 voxels with a narrow key span: the packed dense histogram
fd = (0.5 + rng.random((64, 128, 128)) * 1e-3).astype(np.float32)
check("f32 sorted dense packed", ctx.vcec(torch.from_numpy(fd).cuda()), fd)
# TMA-shaped u8 compute_changes (the bit-sliced kernel's changes mode)
img = rng.integers(0, 9, (10, 40, 48)).astype(np.uint8)
dev = torch.from_numpy(img).cuda()
out = torch.empty(img.size, dtype=torch.int8, device="cuda")
ctx.compute_changes(dev, eb.Dims.of(img.shape), 0, 0, 10, out)
torch.cuda.synchronize()
good = np.array_equal(out.cpu().numpy().reshape(img.shape), oracle.changes(img))
ok &= good
print(("ok  " if good else "BAD ") + "compute_changes u8 TMA-shaped", flush=True)
imgs8 = rng.integers(0, 256, (3, 31, 45)).astype(np.uint8)
chi, pres = ctx.batch2d(imgs8)
t, cc = eb.curve_batch_to_points(chi[1], pres[1])
v, c = oracle.vcec(imgs8[1])
good = np.array_equal(t, v.astype(np.int64)) and np.array_equal(cc, np.cumsum(c))
ok &= good
print(("ok  " if good else "BAD ") + "batch2d u8", flush=True)
# rows of a multiple of 16 bytes: the bit-sliced batch (clusters of several
# CTAs per image for a small batch), packed rows and strips
for shp in ((5, 40, 64), (2, 70, 1024)):
    imgs8 = rng.integers(0, 256, shp).astype(np.uint8)
    chi, pres = ctx.batch2d(imgs8)
    for b in range(shp[0]):
        t, cc = eb.curve_batch_to_points(chi[b], pres[b])
        v, c = oracle.vcec(imgs8[b])
        good = np.array_equal(t, v.astype(np.int64)) and np.array_equal(cc, np.cumsum(c))
        ok &= good
    print(("ok  " if good else "BAD ") + f"batch2d u8 bit-sliced {shp}", flush=True)
img = rng.integers(0, 256, (6, 20, 32)).astype(np.uint8)
dev = torch.from_numpy(img).cuda()
out = torch.empty(img.size, dtype=torch.int8, device="cuda")
ctx.compute_changes(dev, eb.Dims.of(img.shape), 0, 0, 6, out)
torch.cuda.synchronize()
good = np.array_equal(out.cpu().numpy().reshape(img.shape), oracle.changes(img))
ok &= good
print(("ok  " if good else "BAD ") + "compute_changes u8", flush=True)
x = torch.empty((9, 10, 11), dtype=torch.float32, device="cuda")
ctx.uniform_noise(x, seed=2)
y = ctx.gaussian_smooth(x, 2.0, 5)
torch.cuda.synchronize()
good = np.array_equal(y.cpu().numpy().view(np.uint32),
                      oracle.gaussian_smooth(oracle.uniform_noise((9, 10, 11), 2), 2.0, 5).view(np.uint32))
ok &= good
print(("ok  " if good else "BAD ") + "gaussian_smooth", flush=True)
rep = ctx.bench_run(eb.Dims(8, 9, 10), 2)
print("ok  bench_run", rep.last_points, flush=True)
print("ALL OK" if ok else "FAILURES", flush=True)
sys.exit(0 if ok else 1)
