import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle, paper_2203_09087_b200 as eb
ctx = eb.context(0)
rng = np.random.default_rng(3)
def chk(name, img, bm=None):
    a = ctx.vcec(img, binmap=bm) if bm else ctx.vcec(img)
    v, c = oracle.vcec(img)
    print(name, img.shape, np.array_equal(a.changes, c), flush=True)
for lo, hi in [(0, 2), (7, 9), (0, 4)]:
    chk("u16 2D", rng.integers(lo, hi, (4096, 4096)).astype(np.uint16))
    chk("u16 3D", rng.integers(lo, hi, (160, 256, 256)).astype(np.uint16))
    q = (rng.integers(lo, hi, (160, 256, 256)) * 2.0 ** -16).astype(np.float32)
    chk("f32 affine 3D", q, eb.quantised_binmap(65536))
