#!/bin/bash
# Times every variant library under paper_2203_09087_b200/lib/variants with
# the C2 bench line (after a parity check of each through the u8 tests).
TAG=${1:-v}
mkdir -p gpurun_out
for so in paper_2203_09087_b200/lib/variants/*.so; do
  n=$(basename $so .so)
  ECC_B200_LIB=$PWD/$so timeout 300 python -m pytest tests/test_gpu_fast_u8.py -x -q 2>&1 | tail -1 | sed "s/^/$n pytest: /" >> gpurun_out/${TAG}_summary.txt
  for i in 1 2; do
    ECC_B200_LIB=$PWD/$so timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --legs none 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n kernel_ms %.4f frac %.4f' % (d['kernel_ms'], d['roofline']['frac']))" >> gpurun_out/${TAG}_summary.txt
  done
done
cat gpurun_out/${TAG}_summary.txt
