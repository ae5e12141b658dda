"""Device time of large single 2D images through the generic path (probe)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_09087_b200 as eb
ctx = eb.Context(0)
st = torch.cuda.ExternalStream(ctx.stream)
for shape, dt in [((8192, 8192), torch.uint8), ((6400, 3200), torch.uint8), ((8192, 8192), torch.uint16)]:
    img = torch.empty(shape, dtype=dt, device="cuda")
    ctx.fill_synthetic(img, seed=1)
    nb = 256 if dt == torch.uint8 else 65536
    bins = torch.empty(nb, dtype=torch.int32, device="cuda"); chg = torch.empty(nb, dtype=torch.int64, device="cuda")
    chi = torch.empty(nb, dtype=torch.int64, device="cuda"); cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    dims = eb.Dims(shape[0], shape[1], 1)
    for _ in range(3): ctx.curve_device(img, dims, bins, chg, chi, cnt, stream=ctx.stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(10): ctx.curve_device(img, dims, bins, chg, chi, cnt, stream=ctx.stream)
    b.record(st); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(shape, dt, round(ms, 3), "ms", round(img.numel() / ms / 1e6, 1), "GVox/s", flush=True)
# 2D affine-quantised f32 (65536 levels)
img = torch.empty((8192, 8192), dtype=torch.float32, device="cuda")
ctx.fill_synthetic(img, seed=1)
bm = eb.quantised_binmap(65536)
ctx.vcec(img, binmap=bm)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(5): ctx.vcec(img, binmap=bm)
b.record(st); torch.cuda.synchronize()
print("(8192, 8192) f32 affine 65536 vcec (incl. result copy):", round(a.elapsed_time(b) / 5, 3), "ms", flush=True)
