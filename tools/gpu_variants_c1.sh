#!/bin/bash
# C1 + large 2D u8 timing per variant library (u8 2D parity tests first).
TAG=${1:-v1}
mkdir -p gpurun_out
for so in paper_2203_09087_b200/lib/variants/*.so; do
  n=$(basename $so .so)
  ECC_B200_LIB=$PWD/$so timeout 600 python -m pytest tests/test_gpu_u8_2d.py -x -q 2>&1 | tail -1 | sed "s/^/$n pytest: /" >> gpurun_out/${TAG}_summary.txt
  ECC_B200_LIB=$PWD/$so timeout 300 python tools/bench_configs.py C1 2>/dev/null | tail -1 | sed "s/^/$n /" >> gpurun_out/${TAG}_summary.txt
  ECC_B200_LIB=$PWD/$so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_${n}_l.csv python tools/bench_configs.py C1 > /dev/null 2>&1
  python tools/prof_summary.py gpurun_out/${TAG}_${n}_l.csv | grep k_u8_2d | sed "s/^/$n ncu: /" >> gpurun_out/${TAG}_summary.txt
done
cat gpurun_out/${TAG}_summary.txt
