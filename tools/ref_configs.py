"""The reference CPU engine (oracle/_ref, compiled from /root/reference) on
the BASELINE configs, on the host it runs on, for the comparison table in
README.md / DESIGN.md.  Bounded samples; prints one JSON line per config.

  python tools/ref_configs.py > gpurun_out/ref_configs.jsonl
"""
import concurrent.futures as cf
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402

R = oracle.ref()
cores = int(R.ref_hardware_concurrency()) or os.cpu_count()

# C1: best of 20, best reference configuration (1 worker, 1 chunk)
img = oracle.synth("u8", (256, 256))
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    oracle.ref_vcec(img, chunks=1, workers=1)
    ts.append(time.perf_counter() - t0)
print(json.dumps({"config": "C1 256^2 u8", "reference_s": min(ts), "cores": 1,
                  "sample": "best of 20, workers=1 chunks=1"}), flush=True)

# C3: images through the f32 path (u16 values are exact in binary32), one
# image per host thread concurrently (the reference's best configuration)
n = 256
imgs = [oracle.synth("u16", (512, 512), seed=1, base=b * 512 * 512).astype(np.float32)
        for b in range(n)]
t0 = time.perf_counter()
with cf.ThreadPoolExecutor(cores) as ex:
    list(ex.map(lambda a: oracle.ref_vcec(a, chunks=1, workers=1), imgs))
dt = time.perf_counter() - t0
print(json.dumps({"config": "C3 4096 x 512^2 u16 (via the f32 path)",
                  "reference_s_extrapolated": dt * 4096 / n, "measured_images": n,
                  "measured_s": dt, "cores": cores,
                  "sample": f"{n} images, {cores} images in flight, workers=1 chunks=1 each"}),
      flush=True)

# C4: 1024^3 f32 with 65536 levels, CLI-default plan (the radix argsort is
# single-threaded per chunk whatever the worker count)
vol = oracle.synth("f32q", (1024, 1024, 1024))
t0 = time.perf_counter()
oracle.ref_vcec(vol, chunks=max(2, cores), workers=cores)
dt = time.perf_counter() - t0
print(json.dumps({"config": "C4 1024^3 f32 65536 levels", "reference_s": dt, "cores": cores,
                  "sample": f"one pass, workers={cores} chunks={max(2, cores)}"}), flush=True)
