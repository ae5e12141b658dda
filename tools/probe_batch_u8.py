"""Probe: batched 2D u8 images (ctx.batch2d) -- device time of a C3-shaped
u8 batch (4096 x 512^2) and smaller ones, CUDA events on the context stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_09087_b200 as eb  # noqa: E402

ctx = eb.Context(0)
st = torch.cuda.current_stream()  # batch2d runs on torch's current stream
for count, h, w in [(4096, 512, 512), (1024, 256, 256), (64, 1024, 1024)]:
    imgs = torch.randint(0, 256, (count, h, w), dtype=torch.uint8, device="cuda")
    ctx.batch2d(imgs)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(3):
        ctx.batch2d(imgs)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    print({"batch": [count, h, w], "dtype": "u8", "ms": round(ms, 3),
           "gpix_s": round(count * h * w / ms / 1e6, 1)}, flush=True)
