"""Randomised differential test of every public path against the oracle
(test infrastructure): random dtype (u8, u16, f32 from a small pool, f32 on
an affine grid), random 2D / 3D shape (incl. widths around the 32-voxel
chunk and 960-pixel strip edges), random value range (ties, collar-valued
extremes), random path (host / device whole volume, chunked plan, host DMA,
sharded slabs, fused device curve).  Prints one line per failure and a
summary; exits non-zero on any mismatch.

  python tools/fuzz.py [seconds] [seed] [large]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2203_09087_b200 as eb  # noqa: E402
from paper_2203_09087_b200.shard import shard_bounds  # noqa: E402


def grid_values(bm, k):
    """The affine grid exactly as the library defines it (affine_value)."""
    return (np.float64(np.float32(bm["lo"])) + np.asarray(k, np.float64) *
            np.float64(np.float32(bm["step"]))).astype(np.float32)


LARGE = False


def rand_shape(rng):
    if LARGE:
        if rng.random() < 0.4:
            return (int(rng.integers(100, 3000)), int(rng.integers(900, 3000)))
        return (int(rng.integers(20, 200)), int(rng.integers(30, 300)), int(rng.integers(30, 300)))
    if rng.random() < 0.4:
        w = int(rng.choice([1, 2, 31, 32, 33, 63, 64, 65, 959, 960, 961, 1000, int(rng.integers(1, 200))]))
        return (int(rng.integers(1, 70)), w)
    w2 = int(rng.choice([1, 2, 15, 16, 17, 31, 32, 33, 48, 64, int(rng.integers(1, 100))]))
    return (int(rng.integers(1, 40)), int(rng.integers(1, 70)), w2)


def rand_image(rng, shape):
    kind = rng.choice(["u8", "u16", "f32pool", "f32affine", "f32narrow"])
    if kind == "f32narrow":  # general f32 with a narrow key span (the dense path)
        base = np.float32(rng.choice([0.3, 1.0, -2.0, 1000.0]))
        spread = float(rng.choice([2.0 ** -12, 2.0 ** -6, 1.0]))
        img = (base + rng.random(shape) * spread).astype(np.float32)
        if rng.random() < 0.3:
            img = np.round(img * 64) / 64  # ties
        return img.astype(np.float32), None
    if kind == "u8":
        lo, hi = (0, 256) if rng.random() < 0.5 else (int(rng.integers(0, 250)), 256)
        hi = min(256, lo + int(rng.integers(1, 257)))
        return rng.integers(lo, hi, shape).astype(np.uint8), None
    if kind == "u16":
        lo = int(rng.choice([0, 65530, int(rng.integers(0, 65000))]))
        hi = min(65536, lo + int(rng.choice([2, 6, 100, 65536])))
        return rng.integers(lo, hi, shape).astype(np.uint16), None
    if kind == "f32pool":
        pool = np.array([-np.inf, -2.5, -0.0, 0.0, 0.5, 3.0, np.inf], np.float32)
        return pool[rng.integers(0, len(pool), shape)], None
    levels = int(rng.choice([16, 1000, 65536]))
    bm = eb.quantised_binmap(levels)
    # grid values exactly as the library defines them: float32 lo / step,
    # lo + k * step in double, rounded to float32 (ecc_common.cuh affine_value)
    k = rng.integers(0, levels, shape)
    img = (np.float64(np.float32(bm["lo"])) + k * np.float64(np.float32(bm["step"]))).astype(np.float32)
    return img, bm


def run_path(ctx, rng, img, bm):
    path = rng.choice(["host", "device", "plan", "sharded", "curve_device", "batch2d"])
    dims = eb.Dims.of(img.shape)
    if path == "batch2d" and img.ndim == 2 and img.dtype != np.float32:
        chi, pres = ctx.batch2d(img[None])
        t, cc = eb.curve_batch_to_points(chi[0], pres[0].view(np.uint32))
        ch = np.diff(np.concatenate([[0], cc]))
        return path, eb.GlobalVcec(t.astype(img.dtype), ch)
    if path == "batch2d":
        path = "host"
        return path, ctx.vcec(img, binmap=bm)
    if path == "host":
        return path, ctx.vcec(img, binmap=bm)
    if path == "device":
        return path, ctx.vcec(torch.from_numpy(img).cuda(), binmap=bm)
    if path == "plan":
        c = int(rng.integers(1, img.shape[0] + 1))
        plan = eb.plan_chunks(dims, eb.ChunkTarget.count(c), img.dtype)
        return f"plan{c}", eb.process_image(img, plan, binmap=bm)
    if path == "sharded" and img.dtype != np.float32 or (path == "sharded" and bm is not None):
        nb = 256 if img.dtype == np.uint8 else (65536 if img.dtype == np.uint16 else bm["nbins"])
        world = int(rng.integers(1, 4))
        total = torch.zeros(2 * nb, dtype=torch.int64, device="cuda")
        for r in range(world):
            sh = shard_bounds(img.shape[0], world, r)
            if sh.own1 <= sh.own0:
                continue
            slab = torch.from_numpy(np.ascontiguousarray(img[sh.plane0:sh.plane1])).cuda()
            ctx.accumulate_slab(slab, dims, sh.plane0, sh.own0, sh.own1, total, binmap=bm)
        bins = torch.empty(nb, dtype=torch.int32, device="cuda")
        chg = torch.empty(nb, dtype=torch.int64, device="cuda")
        chi = torch.empty(nb, dtype=torch.int64, device="cuda")
        cnt = torch.empty(1, dtype=torch.int64, device="cuda")
        ctx.finalize(total, nb, bins, chg, chi, cnt)
        torch.cuda.synchronize()
        m = int(cnt.item())
        b = bins[:m].cpu().numpy()
        vals = b.astype(img.dtype) if bm is None else grid_values(bm, b)
        return f"sharded{world}", eb.GlobalVcec(vals, chg[:m].cpu().numpy())
    if img.dtype == np.float32 and bm is None:
        return "host", ctx.vcec(img)
    nb = 256 if img.dtype == np.uint8 else (65536 if img.dtype == np.uint16 else bm["nbins"])
    bins = torch.empty(nb, dtype=torch.int32, device="cuda")
    chg = torch.empty(nb, dtype=torch.int64, device="cuda")
    chi = torch.empty(nb, dtype=torch.int64, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    ctx.curve_device(torch.from_numpy(img).cuda(), dims, bins, chg, chi, cnt, binmap=bm)
    torch.cuda.synchronize()
    m = int(cnt.item())
    b = bins[:m].cpu().numpy()
    vals = b.astype(img.dtype) if bm is None else grid_values(bm, b)
    c = chg[:m].cpu().numpy()
    if not np.array_equal(chi[:m].cpu().numpy(), np.cumsum(c)):
        return "curve_device(chi)", eb.GlobalVcec(vals, c * 0 + 10 ** 9)
    return "curve_device", eb.GlobalVcec(vals, c)


def main():
    global LARGE
    seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 120
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    LARGE = len(sys.argv) > 3 and sys.argv[3] == "large"
    rng = np.random.default_rng(seed)
    ctx = eb.context(0)
    t0, n, bad = time.time(), 0, 0
    while time.time() - t0 < seconds:
        shape = rand_shape(rng)
        img, bm = rand_image(rng, shape)
        try:
            path, got = run_path(ctx, rng, img, bm)
        except eb.EccError as e:
            print("ERROR", img.dtype, shape, e, flush=True)
            bad += 1
            n += 1
            continue
        v, c = oracle.vcec(img)
        gv = np.asarray(got.values)
        same_v = (np.array_equal(gv.astype(np.float32).view(np.uint32), np.asarray(v, np.float32).view(np.uint32))
                  if img.dtype == np.float32 else np.array_equal(gv.astype(np.int64), v.astype(np.int64)))
        if not (same_v and np.array_equal(np.asarray(got.changes, np.int64), c)):
            bad += 1
            print("MISMATCH", path, img.dtype, shape, "binmap" if bm else "",
                  "values" if not same_v else "", "changes" if not np.array_equal(
                      np.asarray(got.changes, np.int64), c) else "", flush=True)
        n += 1
    print(f"fuzz: {n} cases, {bad} failures, {time.time() - t0:.0f} s", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
