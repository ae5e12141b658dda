"""Per-config GPU measurements beside bench.py's headline (C2): C1, C3, C4,
C5 (a bounded streamed sample), each checked against its Appendix-B golden
digest (tests/golden/golden.json) before any time is reported.

  python tools/bench_configs.py [C1 C3 C4 C5] > gpurun_out/configs.jsonl

Times are CUDA events on the context stream (device-resident inputs, L2
flushed between reps) unless the line says "e2e" (host buffers, copies
inside).  Not the driver's bench contract -- a development tool whose output
is summarised in profiles/ and DESIGN.md.
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2203_09087_b200 as eb  # noqa: E402

HBM = 6550.4
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["configs"]


def timed(ctx, fn, reps=10, warm=3, flush=None):
    st = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        if flush is not None:
            with torch.cuda.stream(st):
                flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return min(ms), sum(ms) / len(ms)


def digest_of_device_curve(bins, chg, chi, cnt, values_of=None):
    m = int(cnt.item())
    t = bins[:m].cpu().numpy().astype(np.float64)
    if values_of is not None:
        t = values_of(t)
    return oracle.curve_digest(t, chi[:m].cpu().numpy())


def c1(ctx, flush):
    img = torch.from_numpy(oracle.synth("u8", (256, 256))).cuda()
    nb = 256
    bins = torch.empty(nb, dtype=torch.int32, device="cuda")
    chg = torch.empty(nb, dtype=torch.int64, device="cuda")
    chi = torch.empty(nb, dtype=torch.int64, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    dims = eb.Dims(256, 256, 1)
    run = lambda: ctx.curve_device(img, dims, bins, chg, chi, cnt, stream=ctx.stream)
    run()
    torch.cuda.synchronize()
    ok = digest_of_device_curve(bins, chg, chi, cnt) == GOLD["C1"]["digest"]
    best, mean = timed(ctx, run, reps=50, flush=flush)
    host = oracle.synth("u8", (256, 256))
    t0 = time.perf_counter()
    for _ in range(50):
        ctx.curve(host)
    e2e = (time.perf_counter() - t0) / 50
    return {"config": "C1 2D 256^2 u8", "golden": ok, "device_us": mean * 1e3, "best_us": best * 1e3,
            "e2e_us": e2e * 1e6, "gvox_s": 65536 / (mean * 1e-3) / 1e9}


def c3(ctx, flush, count=4096):
    imgs = torch.empty((count, 512, 512), dtype=torch.uint16, device="cuda")
    ctx.fill_synthetic(imgs, seed=1)
    chi = torch.empty((count, 65536), dtype=torch.int32, device="cuda")
    pres = torch.empty((count, 2048), dtype=torch.int32, device="cuda")
    run = lambda: ctx.batch2d(imgs, chi=chi, presence=pres, stream=ctx.stream)
    run()
    torch.cuda.synchronize()
    ok = True
    for b in (0, count - 1) if count == 4096 else ():
        t, cc = eb.curve_batch_to_points(chi[b].cpu().numpy(), pres[b].cpu().numpy().view(np.uint32))
        ok &= oracle.curve_digest(t, cc) == GOLD[f"C3_{b}"]["digest"]
    best, mean = timed(ctx, run, reps=5, flush=flush)
    vox = count * 512 * 512
    alg = vox * 2 + count * 65536 * 4 + count * 65536 // 8
    return {"config": f"C3 {count} x 512^2 u16 batched", "golden": ok, "device_ms": mean,
            "best_ms": best, "gvox_s": vox / (mean * 1e-3) / 1e9,
            "hbm_frac": alg / (mean * 1e-3) / 1e9 / HBM}


def c4(ctx, flush, side=1024):
    vol = torch.empty((side, side, side), dtype=torch.float32, device="cuda")
    ctx.fill_synthetic(vol, seed=1)
    nb = 65536
    bins = torch.empty(nb, dtype=torch.int32, device="cuda")
    chg = torch.empty(nb, dtype=torch.int64, device="cuda")
    chi = torch.empty(nb, dtype=torch.int64, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    dims = eb.Dims(side, side, side)
    bm = eb.quantised_binmap(65536)
    run = lambda: ctx.curve_device(vol, dims, bins, chg, chi, cnt, binmap=bm, stream=ctx.stream)
    run()
    torch.cuda.synchronize()
    ok = digest_of_device_curve(bins, chg, chi, cnt, values_of=lambda t: t * 2.0 ** -16) == \
        GOLD["C4"]["digest"] if side == 1024 else None
    best, mean = timed(ctx, run, reps=5, flush=flush)
    vox = side ** 3
    return {"config": f"C4 {side}^3 f32 65536 levels", "golden": ok, "device_ms": mean,
            "best_ms": best, "gvox_s": vox / (mean * 1e-3) / 1e9,
            "hbm_frac": vox * 4 / (mean * 1e-3) / 1e9 / HBM}


def c5(ctx, planes=256, chunk=32):
    """Streams the first `planes` planes of the 4096^3 u8 volume from pinned
    host memory through ecc_process_host (chunk-plane slabs + halo, DMA
    straight from the pinned buffer, 3 device buffers in flight).  The first
    64 planes are checked against the Appendix-B golden."""
    side = 4096
    host = torch.empty((planes, side, side), dtype=torch.uint8, pin_memory=True)
    step = 64
    for a in range(0, planes, step):  # fill in 1 GiB pieces on the GPU
        dev = torch.empty((min(step, planes - a), side, side), dtype=torch.uint8, device="cuda")
        ctx.fill_synthetic(dev, seed=1, base=a * side * side)
        host[a:a + dev.shape[0]].copy_(dev)
        del dev
    torch.cuda.synchronize()
    arr = host.numpy()
    a64 = arr[:64]
    v = ctx.process_host(a64, eb.plan_chunks(eb.Dims(64, side, side), eb.ChunkTarget.count(4)))
    cur = eb.vcec_to_ecc(v)
    ok = oracle.curve_digest(cur.thresholds.astype(np.float64), cur.chi) == GOLD["C5_64"]["digest"]
    plan = eb.plan_chunks(eb.Dims(planes, side, side), eb.ChunkTarget.count(planes // chunk))
    ctx.process_host(arr, plan)
    reps = 3 if planes <= 512 else 1
    t0 = time.perf_counter()
    rep = eb.EngineReport()
    for _ in range(reps):
        v = ctx.process_host(arr, plan, report=rep)
    dt = (time.perf_counter() - t0) / reps
    assert v.total() == 1
    vox = planes * side * side
    h2d = sum(c.ingest_end - c.ingest_begin for c in rep.chunks)
    kern = sum(c.kernel_end - c.kernel_begin for c in rep.chunks)
    moved = sum((min(c.range.end + 1, planes) - max(c.range.begin - 1, 0)) for c in rep.chunks) * side * side
    return {"config": f"C5 first {planes} planes of 4096^3 u8, streamed from pinned host (e2e)",
            "golden_first_64": ok, "e2e_ms": dt * 1e3, "gvox_s": vox / dt / 1e9,
            "h2d_gb_s_during_copies": moved / h2d / 1e9, "h2d_busy_s": h2d, "kernel_busy_s": kern,
            "chunks": len(rep.chunks)}


if __name__ == "__main__":
    which = sys.argv[1:] or ["C1", "C3", "C4", "C5"]
    ctx = eb.Context(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for w in which:
        try:
            r = {"C1": lambda: c1(ctx, flush), "C3": lambda: c3(ctx, flush),
                 "C4": lambda: c4(ctx, flush), "C5": lambda: c5(ctx),
                 "C5full": lambda: c5(ctx, planes=4096, chunk=128)}[w]()
        except Exception as e:  # report and continue with the next config
            r = {"config": w, "error": repr(e)[:300]}
        print(json.dumps(r), flush=True)
        torch.cuda.empty_cache()
