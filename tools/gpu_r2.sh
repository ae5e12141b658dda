#!/bin/bash
# Round-2 GPU check: new tests + the bench line (with the C4 / C5 legs).
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
free -g >> gpurun_out/${TAG}_smi.txt; nproc >> gpurun_out/${TAG}_smi.txt
timeout 900 python -m pytest tests/test_gpu_round2.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -3 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_bench.json; tail -5 gpurun_out/${TAG}_bench.err
