#!/bin/bash
# Large single 2D images + C1 per variant library (u8 2D parity tests first).
TAG=${1:-v2d}
mkdir -p gpurun_out
for so in paper_2203_09087_b200/lib/variants/*.so; do
  n=$(basename $so .so)
  ECC_B200_LIB=$PWD/$so timeout 600 python -m pytest tests/test_gpu_u8_2d.py tests/test_gpu_parity.py -x -q -k "u8 or config1 or 2d" 2>&1 | tail -1 | sed "s/^/$n pytest: /" >> gpurun_out/${TAG}_summary.txt
  ECC_B200_LIB=$PWD/$so timeout 300 python tools/probe_2d.py 2>/dev/null | head -2 | sed "s/^/$n /" >> gpurun_out/${TAG}_summary.txt
  ECC_B200_LIB=$PWD/$so timeout 300 python tools/bench_configs.py C1 2>/dev/null | tail -1 | sed "s/^/$n /" >> gpurun_out/${TAG}_summary.txt
done
cat gpurun_out/${TAG}_summary.txt
