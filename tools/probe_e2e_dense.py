"""End to end from pinned host memory for the dense maps (overlapped path):
a 512 x 1024 x 1024 quantised f32 volume (2 GiB) and a 1024 x 512 x 512
u16 volume, against the bare H2D copy."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_09087_b200 as eb
ctx = eb.context(0)
for shape, dt, bm in [((512, 1024, 1024), torch.float32, eb.quantised_binmap(65536)),
                      ((1024, 512, 512), torch.uint16, None)]:
    dev = torch.empty(shape, dtype=dt, device="cuda")
    ctx.fill_synthetic(dev, seed=1)
    host = torch.empty(shape, dtype=dt, pin_memory=True)
    host.copy_(dev)
    arr = host.numpy()
    for _ in range(2): ctx.vcec(arr, binmap=bm) if bm else ctx.vcec(arr)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ctx.vcec(arr, binmap=bm) if bm else ctx.vcec(arr)
        ts.append(time.perf_counter() - t0)
    h = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter(); dev.copy_(host, non_blocking=True); torch.cuda.synchronize(); h.append(time.perf_counter() - t0)
    print(shape, dt, "e2e %.2f ms, bare H2D %.2f ms" % (1e3 * min(ts), 1e3 * min(h)), flush=True)
    del dev, host
