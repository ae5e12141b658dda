import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle, paper_2203_09087_b200 as eb
ctx = eb.context(0)
rng = np.random.default_rng(1)
for lo, hi in [(0, 2), (65530, 65536), (1000, 1006), (0, 100)]:
    for shape in [(2035, 1197), (300, 1100), (2000, 1024), (2000, 512)]:
        img = rng.integers(lo, hi, shape).astype(np.uint16)
        chi, pres = ctx.batch2d(img[None])
        t, cc = eb.curve_batch_to_points(chi[0], pres[0].view(np.uint32))
        v, c = oracle.vcec(img)
        ok_t = np.array_equal(t, v.astype(np.int64)); ok_c = ok_t and np.array_equal(cc, np.cumsum(c))
        print((lo, hi), shape, ok_t, ok_c, "" if ok_c else (cc[:4], np.cumsum(c)[:4]), flush=True)
