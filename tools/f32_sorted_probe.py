"""Probe: general (sorted-distinct) f32 path on uniform random 256^3 / 512^3
volumes -- wall time of ctx.vcec and parity against the oracle."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2203_09087_b200 as eb, oracle
ctx = eb.Context(0)
for side in (256, 512):
    rng = np.random.default_rng(1)
    img = rng.random((side, side, side), dtype=np.float32)
    ctx.vcec(img[:8])  # warm
    t0 = time.perf_counter(); v = ctx.vcec(img); t1 = time.perf_counter()
    plan = eb.plan_chunks(eb.Dims.of(img.shape), eb.ChunkTarget.count(8))
    t2 = time.perf_counter(); w = eb.process_image(img, plan); t3 = time.perf_counter()
    print(side, "whole", round(t1 - t0, 3), "s; 8 chunks", round(t3 - t2, 3), "s; values", v.size(), "same", np.array_equal(v.changes, w.changes), flush=True)
    if side == 256:
        t4 = time.perf_counter(); r = oracle.ref_vcec(img, chunks=16, workers=16); t5 = time.perf_counter()
        print(" ref", round(t5 - t4, 3), "s", np.array_equal(r[1], v.changes), flush=True)
