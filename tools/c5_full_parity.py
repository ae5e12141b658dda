"""C5 end to end: the full 4096^3 u8 synthetic volume (64 GiB, SURVEY.md
8(d): v = counter_hash(1, i) >> 56) streamed from pinned host memory through
ecc_process_host on one B200, checked bit-exactly against the UNMODIFIED
reference engine (oracle/_ref, compiled from /root/reference) run on the
same host buffer with all host threads.  Writes one JSON line.

  python tools/c5_full_parity.py [planes] > gpurun_out/c5_parity.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2203_09087_b200 as eb  # noqa: E402

planes = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
side = 4096
ctx = eb.Context(0)
host = torch.empty((planes, side, side), dtype=torch.uint8, pin_memory=True)
for a in range(0, planes, 64):
    dev = torch.empty((min(64, planes - a), side, side), dtype=torch.uint8, device="cuda")
    ctx.fill_synthetic(dev, seed=1, base=a * side * side)
    host[a:a + dev.shape[0]].copy_(dev)
    del dev
torch.cuda.synchronize()
arr = host.numpy()
plan = eb.plan_chunks(eb.Dims(planes, side, side), eb.ChunkTarget.count(max(1, planes // 128)))
t0 = time.perf_counter()
ours = ctx.process_host(arr, plan)
t_ours = time.perf_counter() - t0
R = oracle.ref()
cores = int(R.ref_hardware_concurrency()) or os.cpu_count()
t0 = time.perf_counter()
rv, rc = oracle.ref_vcec(arr, chunks=max(2, planes // 64), workers=cores)
t_ref = time.perf_counter() - t0
same = bool(np.array_equal(ours.values.astype(np.int64), rv.astype(np.int64)) and
            np.array_equal(ours.changes, rc))
chi = np.cumsum(ours.changes)
print(json.dumps({"config": f"C5 {planes}x{side}x{side} u8 streamed from pinned host",
                  "bit_exact_vs_reference": same, "points": int(len(chi)),
                  "final_chi": int(chi[-1]), "min_chi": int(chi.min()), "max_chi": int(chi.max()),
                  "ours_s": t_ours, "ours_gvox_s": planes * side * side / t_ours / 1e9,
                  "reference_s": t_ref, "reference_cores": cores,
                  "reference_gvox_s": planes * side * side / t_ref / 1e9,
                  "digest": oracle.curve_digest(ours.values.astype(np.float64), chi)}), flush=True)
