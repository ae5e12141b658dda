"""Wall time of host-returning general-f32 calls (ctx.vcec on a device
volume): the GPU part is ~1 ms, the rest is result handling on the host."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_09087_b200 as eb  # noqa: E402

ctx = eb.Context(0)
S = 512
vol = torch.empty((S, S, S), dtype=torch.float32, device="cuda")
ctx.uniform_noise(vol, seed=1, stream=ctx.stream)
sm = torch.empty_like(vol)
ctx.gaussian_smooth(vol, 2.0, 13, out=sm, stream=ctx.stream)
torch.cuda.synchronize()
ts = []
for i in range(6):
    t0 = time.perf_counter()
    r = ctx.vcec(sm)
    ts.append((time.perf_counter() - t0) * 1e3)
print({"case": "vcec 512^3 smoothed f32 (device input, host result)", "points": r.size(),
       "wall_ms": [round(t, 2) for t in ts]})
