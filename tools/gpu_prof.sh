#!/bin/bash
# One ncu --set full capture of the u8 3D kernel under the bench (1 GPU),
# plus the raw metrics and source pages exported next to it.
TAG=${1:-p}
KREGEX=${2:-k_u8_3d}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s 2 -c 1 -o gpurun_out/${TAG}_prof \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --legs none > gpurun_out/${TAG}_ncu.log 2>&1
tail -1 gpurun_out/${TAG}_ncu.log
ncu -i gpurun_out/${TAG}_prof.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_prof.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
ls -la gpurun_out/${TAG}_*
