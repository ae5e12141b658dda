#!/bin/bash
# One ncu --set full capture of a kernel under tools/bench_configs.py <config>
# (1 GPU), plus the raw metrics and SASS source pages next to it.
#   bash tools/gpu_prof_cfg.sh <tag> <config> <kernel regex>
TAG=${1:-pc}
CFG=${2:-C3}
KREGEX=${3:-k_batch16}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s 1 -c 1 -o gpurun_out/${TAG}_prof \
  python tools/bench_configs.py ${CFG} > gpurun_out/${TAG}_ncu.log 2>&1
tail -1 gpurun_out/${TAG}_ncu.log
ncu -i gpurun_out/${TAG}_prof.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_prof.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
ls -la gpurun_out/${TAG}_*
