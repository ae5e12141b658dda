"""Device time of gaussian_smooth (3 axes, width 13) on 512^3 f32, and of bench_run."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_09087_b200 as eb
ctx = eb.Context(0)
st = torch.cuda.ExternalStream(ctx.stream)
x = torch.empty((512, 512, 512), dtype=torch.float32, device="cuda")
ctx.uniform_noise(x, seed=1)
y = torch.empty_like(x)
for _ in range(2): ctx.gaussian_smooth(x, 2.0, 13, out=y, stream=ctx.stream)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(5): ctx.gaussian_smooth(x, 2.0, 13, out=y, stream=ctx.stream)
b.record(st); torch.cuda.synchronize()
print("smooth 512^3 w13:", round(a.elapsed_time(b) / 5, 3), "ms", flush=True)
for _ in range(3):
    r = ctx.bench_run(eb.Dims(512, 512, 512), 3)
    print("bench_run: smooth", round(r.smooth_avg_s * 1e3, 2), "ms, ecc", round(r.ecc_avg_s * 1e3, 2), "ms", flush=True)
# the general-f32 curve of the smoothed volume through ecc_vcec (dense key
# histogram when the key span allows), device time of the whole call
import time
y = ctx.gaussian_smooth(x, 2.0, 13)
torch.cuda.synchronize()
for _ in range(2): ctx.vcec(y)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5): v = ctx.vcec(y)
t1 = time.perf_counter()
print("vcec smoothed 512^3 (dense path if the key span allows):", round((t1 - t0) / 5 * 1e3, 2), "ms;", v.size(), "values", flush=True)
