import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
buf = torch.zeros(4 * 8 * 32 * 12, dtype=torch.int32, device="cuda")
os.environ["ECC_DBG_PTR"] = str(buf.data_ptr())
import paper_2203_09087_b200 as eb
ctx = eb.Context(0)
rng = np.random.default_rng(0)
shape = (3, 30, 32)
img = rng.integers(0, 256, shape).astype(np.uint8)
dev = torch.from_numpy(img).cuda()
out = torch.full(shape, 99, dtype=torch.int8, device="cuda")
ctx.compute_changes(dev, eb.Dims.of(shape), 0, 0, shape[0], out)
torch.cuda.synchronize()
np.save("gpurun_out/dbg_win.npy", buf.cpu().numpy().view(np.uint32).reshape(4, 8, 32, 12))
print("ok")
