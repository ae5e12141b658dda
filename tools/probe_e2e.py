"""C2 end to end from pinned host memory: one-shot ecc_curve vs the chunked
host-DMA driver (ecc_process_host) at several chunk counts."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_09087_b200 as eb
ctx = eb.context(0)
dev = torch.empty((512, 512, 512), dtype=torch.uint8, device="cuda")
ctx.fill_synthetic(dev, seed=1)
host = torch.empty((512, 512, 512), dtype=torch.uint8, pin_memory=True)
host.copy_(dev.cpu())
arr = host.numpy()
def t(fn, reps=20):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return 1e3 * sum(ts) / len(ts), 1e3 * min(ts)
print("curve (one shot):", t(lambda: ctx.curve(arr)), flush=True)
for c in (2, 4, 8, 16):
    plan = eb.plan_chunks(eb.Dims.of(arr.shape), eb.ChunkTarget.count(c), np.uint8)
    print(f"process_host {c} chunks:", t(lambda: ctx.process_host(arr, plan)), flush=True)
h2d = torch.empty_like(dev)
print("plain H2D copy:", t(lambda: (h2d.copy_(host, non_blocking=True), torch.cuda.synchronize())), flush=True)
