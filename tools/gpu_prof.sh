#!/bin/bash
# One ncu --set full capture of the u8 3D kernel under the bench (1 GPU).
TAG=${1:-p}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_u8_3d -s 2 -c 1 -o gpurun_out/${TAG}_prof \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
tail -1 gpurun_out/${TAG}_ncu.log
