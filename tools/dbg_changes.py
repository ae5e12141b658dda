import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2203_09087_b200 as eb
ctx = eb.Context(0)
rng = np.random.default_rng(0)
shape = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (3, 30, 32)
img = rng.integers(0, 256, shape).astype(np.uint8)
dev = torch.from_numpy(img).cuda()
out = torch.full(shape, 99, dtype=torch.int8, device="cuda")
ctx.compute_changes(dev, eb.Dims.of(shape), 0, 0, shape[0], out)
torch.cuda.synchronize()
got = out.cpu().numpy().astype(np.int64)
want = oracle.changes(img).reshape(shape).astype(np.int64)
bad = np.argwhere(got != want)
print("mismatches", len(bad), "of", got.size)
for b in bad[:40]:
    print(tuple(b), "got", got[tuple(b)], "want", want[tuple(b)])
np.save("gpurun_out/dbg_got.npy", got)
