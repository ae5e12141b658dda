import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, json
import oracle, paper_2203_09087_b200 as eb
ctx = eb.Context(0)
dev = torch.empty((64, 4096, 4096), dtype=torch.uint8, device="cuda")
ctx.fill_synthetic(dev, seed=1)
c = ctx.curve(dev)
print(len(c.thresholds), c.thresholds[0], c.chi[0], c.chi[-1], c.chi.min(), c.chi.max())
print(oracle.curve_digest(c.thresholds.astype(np.float64), c.chi))
host = oracle.synth("u8", (64, 4096, 4096))
print("gen equal", np.array_equal(host, dev.cpu().numpy()))
