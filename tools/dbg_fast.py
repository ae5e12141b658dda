import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle, paper_2203_09087_b200 as eb
ctx = eb.Context(0)
rng = np.random.default_rng(0)
shape = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (3, 30, 32)
img = rng.integers(0, 256, shape).astype(np.uint8)
a = ctx.vcec(img)
v, c = oracle.vcec(img)
print("values ok", np.array_equal(a.values.astype(np.int64), v.astype(np.int64)), "changes ok", np.array_equal(a.changes, c))
print(a.changes[:10], c[:10])
