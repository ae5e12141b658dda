#!/bin/bash
# C3 timing (golden-checked by bench_configs) + the batched parity tests per variant library.
TAG=${1:-v3}
mkdir -p gpurun_out
for so in paper_2203_09087_b200/lib/variants/*.so; do
  n=$(basename $so .so)
  ECC_B200_LIB=$PWD/$so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_u16_2d.py -x -q -k "batch or config3 or hot" 2>&1 | tail -1 | sed "s/^/$n pytest: /" >> gpurun_out/${TAG}_summary.txt
  ECC_B200_LIB=$PWD/$so timeout 600 python tools/bench_configs.py C3 2>/dev/null | tail -1 | sed "s/^/$n /" >> gpurun_out/${TAG}_summary.txt
done
cat gpurun_out/${TAG}_summary.txt
