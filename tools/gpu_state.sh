#!/bin/bash
# Where every config stands: golden-checked C1/C3/C4 device times, large 2D
# images, the smoothing + ECC pipeline, and the C1 launch list under ncu.
TAG=${1:-s}
mkdir -p gpurun_out
timeout 900 python tools/bench_configs.py C1 C3 C4 > gpurun_out/${TAG}_configs.jsonl 2> gpurun_out/${TAG}_configs.err
timeout 300 python tools/probe_2d.py > gpurun_out/${TAG}_2d.txt 2>&1
timeout 600 python tools/bench_pipeline.py 512 5 0 > gpurun_out/${TAG}_pipeline.jsonl 2>&1
timeout 300 python tools/probe_generic.py > gpurun_out/${TAG}_generic.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c1_launches.csv \
  python tools/bench_configs.py C1 > /dev/null 2>&1
cat gpurun_out/${TAG}_configs.jsonl gpurun_out/${TAG}_2d.txt gpurun_out/${TAG}_pipeline.jsonl gpurun_out/${TAG}_generic.jsonl
grep -o '"k_[a-z0-9_]*[^"]*","[^"]*","[^"]*"' gpurun_out/${TAG}_c1_launches.csv | head -0
python tools/prof_summary.py gpurun_out/${TAG}_c1_launches.csv | head -12
