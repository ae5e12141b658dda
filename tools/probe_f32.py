"""Device-side cost of the general (sorted) f32 path on a resident 512^3
random f32 volume: compute_changes alone, and the whole curve."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_09087_b200 as eb
ctx = eb.Context(0)
st = torch.cuda.ExternalStream(ctx.stream)
n = 512
img = torch.empty((n, n, n), dtype=torch.float32, device="cuda")
ctx.fill_synthetic(img, seed=1)
dims = eb.Dims(n, n, n)
out = torch.empty(n ** 3, dtype=torch.int8, device="cuda")
for _ in range(2):
    ctx.compute_changes(img, dims, 0, 0, n, out, stream=ctx.stream)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(5):
    ctx.compute_changes(img, dims, 0, 0, n, out, stream=ctx.stream)
b.record(st); torch.cuda.synchronize()
print("compute_changes f32 512^3:", round(a.elapsed_time(b) / 5, 3), "ms", flush=True)
for _ in range(2):
    ctx.vcec(img)
torch.cuda.synchronize()
t0 = time.perf_counter()
v = ctx.vcec(img)
t1 = time.perf_counter()
print("vcec f32 512^3 (device input, host result):", round((t1 - t0) * 1e3, 1), "ms; values", v.size(), flush=True)
