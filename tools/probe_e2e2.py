"""Probe: end-to-end C2 (512^3 u8 from pinned host memory) through the
Python API, the overlapped H2D + kernel path, against the device-resident time."""
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
ts = []
for i in range(40):
    torch.cuda.synchronize(); t0 = time.perf_counter(); ctx.curve(arr); ts.append(time.perf_counter() - t0)
ts = ts[5:]
print(os.environ.get("ECC_B200_OVERLAP_CHUNKS"), "mean %.3f min %.3f median %.3f p90 %.3f max %.3f ms" % (1e3*np.mean(ts), 1e3*min(ts), 1e3*np.median(ts), 1e3*np.percentile(ts, 90), 1e3*max(ts)), flush=True)
h2d = torch.empty_like(dev)
ts = []
for i in range(40):
    torch.cuda.synchronize(); t0 = time.perf_counter(); h2d.copy_(host, non_blocking=True); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
ts = ts[5:]
print("H2D only: mean %.3f min %.3f median %.3f p90 %.3f max %.3f ms" % (1e3*np.mean(ts), 1e3*min(ts), 1e3*np.median(ts), 1e3*np.percentile(ts, 90), 1e3*max(ts)), flush=True)
