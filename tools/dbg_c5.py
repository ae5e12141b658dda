import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, json
import oracle, paper_2203_09087_b200 as eb
ctx = eb.Context(0)
rng = np.random.default_rng(0)
for shape, chunks in [((20, 100, 128), 3), ((64, 64, 64), 4), ((16, 512, 512), 2), ((40, 1000, 992), 4)]:
    img = rng.integers(0, 256, shape).astype(np.uint8)
    want = oracle.vcec(img)
    a = ctx.vcec(img)
    plan = eb.plan_chunks(eb.Dims.of(shape), eb.ChunkTarget.count(chunks))
    b = eb.process_image(img, plan)
    print(shape, chunks, "whole", np.array_equal(a.changes, want[1]), "stream", np.array_equal(b.changes, want[1]), flush=True)
for planes in (16, 32, 64):
    side = 4096
    dev = torch.empty((planes, side, side), dtype=torch.uint8, device="cuda")
    ctx.fill_synthetic(dev, seed=1)
    a = ctx.vcec(dev)
    arr = dev.cpu().numpy()
    h, c = oracle.hist_dense(arr) if planes <= 16 else (None, None)
    plan = eb.plan_chunks(eb.Dims(planes, side, side), eb.ChunkTarget.count(max(1, planes // 16)))
    b = eb.process_image(arr, plan)
    print(planes, "whole==stream", np.array_equal(a.changes, b.changes), a.total(), b.total(),
          "oracle" if h is None else np.array_equal(a.changes, h[c > 0]), flush=True)
