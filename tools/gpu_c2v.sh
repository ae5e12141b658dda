#!/bin/bash
# C2 variant check: u8 3D parity tests, parity suite, short fuzz, two C2 bench lines.
TAG=${1:-c2v}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast_u8.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 150 python tools/fuzz.py 90 7 > gpurun_out/${TAG}_fuzz_small.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_fuzz_small.log
timeout 150 python tools/fuzz.py 90 8 large > gpurun_out/${TAG}_fuzz_large.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_fuzz_large.log
for i in 1 2; do timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --legs none 2>>gpurun_out/${TAG}_bench.err | tail -1 >> gpurun_out/${TAG}_bench.json; done
timeout 120 python tools/probe_3d_sizes.py > gpurun_out/${TAG}_sizes.txt 2>&1
tail -2 gpurun_out/${TAG}_pytest.log; tail -3 gpurun_out/${TAG}_fuzz_small.log gpurun_out/${TAG}_fuzz_large.log; cat gpurun_out/${TAG}_sizes.txt | tail -8
python - <<PY
import json
for l in open("gpurun_out/${TAG}_bench.json"):
    d=json.loads(l); print("kernel_ms %.4f frac %.4f e2e %.1f GVox/s value %.1f golden %s" % (d["kernel_ms"], d["roofline"]["frac"], d["e2e"]["value"], d["value"], d.get("checks")))
PY
