#!/bin/bash
# C2 iteration loop: u8 3D parity tests + the C2 bench line (no legs, no CPU arm).
TAG=${1:-c2}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fast_u8.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for i in 1 2; do timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --legs none 2>>gpurun_out/${TAG}_bench.err | tail -1 >> gpurun_out/${TAG}_bench.json; done
tail -2 gpurun_out/${TAG}_pytest.log
python - <<PY
import json
for l in open("gpurun_out/${TAG}_bench.json"):
    d=json.loads(l); print("kernel_ms %.4f frac %.4f e2e %.1f GVox/s value %.1f" % (d["kernel_ms"], d["roofline"]["frac"], d["e2e"]["value"], d["value"]))
PY
