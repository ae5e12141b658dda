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
