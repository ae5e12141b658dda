"""Probe: single 2D u16 images of moderate size through curve_device
(k_u16_2d: one CTA per SM, each flushing a 65536-bin table) -- device time
by CUDA events on the context stream, with the launch list in mind."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_09087_b200 as eb  # noqa: E402

ctx = eb.Context(0)
st = torch.cuda.ExternalStream(ctx.stream)
for shape in [(512, 512), (1024, 1024), (2048, 2048), (4096, 4096)]:
    img = torch.randint(0, 65536, shape, dtype=torch.int32, device="cuda").to(torch.uint16)
    nb = 65536
    bins = torch.empty(nb, dtype=torch.int32, device="cuda")
    chg = torch.empty(nb, dtype=torch.int64, device="cuda")
    chi = torch.empty(nb, dtype=torch.int64, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    dims = eb.Dims(shape[0], shape[1], 1)
    for _ in range(3):
        ctx.curve_device(img, dims, bins, chg, chi, cnt, stream=ctx.stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(10):
        ctx.curve_device(img, dims, bins, chg, chi, cnt, stream=ctx.stream)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print({"shape": shape, "dtype": "u16", "us": round(ms * 1e3, 1),
           "gpix_s": round(shape[0] * shape[1] / ms / 1e6, 1)}, flush=True)
