"""bench_run (pipeline.hpp:236-291) on the GPU beside the reference's own
bench_run on the host cores, same dims / iterations / sigma / width.

  python tools/bench_pipeline.py [side] [iterations] [ref_side]   (ref_side 0: GPU only)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2203_09087_b200 as eb  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 512
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ref_side = int(sys.argv[3]) if len(sys.argv) > 3 else 128
ctx = eb.context(0)
ctx.bench_run(eb.Dims(side, side, side), 1)  # warm-up at the same size (allocations, module load)
rep = ctx.bench_run(eb.Dims(side, side, side), iters)
out = {"impl": "b200", "dims": [side] * 3, **rep.__dict__}
print(json.dumps(out), flush=True)
if ref_side > 0 and oracle.ref_available():
    r = oracle.ref_bench_run((ref_side,) * 3, 1)
    print(json.dumps({"impl": "reference (host cores)", "dims": [ref_side] * 3, "iterations": 1, **r}),
          flush=True)
