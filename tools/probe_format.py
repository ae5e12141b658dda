"""Device time of ecc_batch_format on the C3 batch (4096 x 512^2 u16)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_09087_b200 as eb
ctx = eb.context(0)
imgs = torch.empty((4096, 512, 512), dtype=torch.uint16, device="cuda")
ctx.fill_synthetic(imgs, seed=1)
chi, pres = ctx.batch2d(imgs)
torch.cuda.synchronize()
for fmt in ("csv", "json"):
    ctx.batch_format(chi, pres, np.uint16, fmt)
    t0 = time.perf_counter(); files = ctx.batch_format(chi, pres, np.uint16, fmt); t1 = time.perf_counter()
    print(fmt, "4096 curves,", sum(map(len, files)) / 1e9, "GB, whole call incl. D2H + split:", round(t1 - t0, 3), "s", flush=True)
