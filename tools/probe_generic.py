"""Timing probe of the generic (tournament) kernels: 512^3 f32 compute_changes,
the whole-volume general-f32 ECC of a smoothed field (dense key histogram),
a ragged u8 volume and a 2D f32 image.  Device time by CUDA events on the
context stream; prints one JSON line per case."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_09087_b200 as eb  # noqa: E402

ctx = eb.Context(0)
st = torch.cuda.ExternalStream(ctx.stream)


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), sorted(ts)[len(ts) // 2]


S = 512
vol = torch.empty((S, S, S), dtype=torch.float32, device="cuda")
ctx.uniform_noise(vol, seed=1, stream=ctx.stream)
sm = torch.empty_like(vol)
ctx.gaussian_smooth(vol, 2.0, 13, out=sm, stream=ctx.stream)
torch.cuda.synchronize()
dims = eb.Dims(S, S, S)
chg = torch.empty((S, S, S), dtype=torch.int8, device="cuda")
best, med = timed(lambda: ctx.compute_changes(vol, dims, 0, 0, S, chg, stream=ctx.stream))
print(json.dumps({"case": "compute_changes 512^3 f32", "ms_best": best, "ms_median": med,
                  "GBps": S ** 3 * 4 / best / 1e6}), flush=True)
res = {}
best, med = timed(lambda: res.setdefault("v", ctx.vcec(sm)), reps=5)
print(json.dumps({"case": "vcec 512^3 smoothed f32 (sorted map, incl. D2H)", "ms_best": best,
                  "ms_median": med, "points": int(res["v"].size())}), flush=True)
rag = torch.randint(0, 256, (301, 299, 297), dtype=torch.uint8, device="cuda")
hist = torch.zeros(512, dtype=torch.int64, device="cuda")
d2 = eb.Dims(301, 299, 297)
best, med = timed(lambda: ctx.accumulate_slab(rag, d2, 0, 0, 301, hist, stream=ctx.stream))
print(json.dumps({"case": "accumulate ragged 301x299x297 u8", "ms_best": best, "ms_median": med,
                  "GVoxps": 301 * 299 * 297 / best / 1e6}), flush=True)
img = torch.rand((4096, 4096, 1), device="cuda")
d3 = eb.Dims(4096, 4096, 1)
c2 = torch.empty((4096, 4096), dtype=torch.int8, device="cuda")
best, med = timed(lambda: ctx.compute_changes(img, d3, 0, 0, 4096, c2, stream=ctx.stream))
print(json.dumps({"case": "compute_changes 4096^2 f32 2D", "ms_best": best, "ms_median": med,
                  "GBps": 4096 * 4096 * 4 / best / 1e6}), flush=True)
