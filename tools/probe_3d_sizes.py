"""Probe: single 3D u8 / u16 volumes of several sizes through curve_device
(one fused launch for u8) -- device time per call, CUDA events on the
context stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_09087_b200 as eb  # noqa: E402

ctx = eb.Context(0)
st = torch.cuda.ExternalStream(ctx.stream)
for dt, nb in ((torch.uint8, 256), (torch.uint16, 65536)):
    for side in (32, 64, 128, 256, 512):
        hi = 256 if dt == torch.uint8 else 65536
        img = torch.randint(0, hi, (side, side, side), dtype=torch.int32, device="cuda").to(dt)
        bins = torch.empty(nb, dtype=torch.int32, device="cuda")
        chg = torch.empty(nb, dtype=torch.int64, device="cuda")
        chi = torch.empty(nb, dtype=torch.int64, device="cuda")
        cnt = torch.empty(1, dtype=torch.int64, device="cuda")
        dims = eb.Dims(side, side, side)
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
        print({"side": side, "dtype": str(dt).split(".")[-1], "us": round(ms * 1e3, 1),
               "gvox_s": round(side ** 3 / ms / 1e6, 1)}, flush=True)
