#!/bin/bash
# u16 3D kernel check: parity tests, short fuzz, per-size device times, C4 golden-checked time.
TAG=${1:-u16v}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 150 python tools/fuzz.py 90 17 > gpurun_out/${TAG}_fuzz_small.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_fuzz_small.log
timeout 150 python tools/fuzz.py 90 18 large > gpurun_out/${TAG}_fuzz_large.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_fuzz_large.log
timeout 120 python tools/probe_3d_sizes.py > gpurun_out/${TAG}_sizes.txt 2>&1
timeout 600 python tools/bench_configs.py C4 > gpurun_out/${TAG}_c4.jsonl 2> gpurun_out/${TAG}_c4.err
tail -2 gpurun_out/${TAG}_pytest.log; tail -2 gpurun_out/${TAG}_fuzz_small.log gpurun_out/${TAG}_fuzz_large.log; cat gpurun_out/${TAG}_sizes.txt gpurun_out/${TAG}_c4.jsonl | cut -c1-300
