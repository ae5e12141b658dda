#!/bin/bash
# C4 timing (bench leg, golden-checked) + the u16 parity tests per variant library.
TAG=${1:-v4}
mkdir -p gpurun_out
for so in paper_2203_09087_b200/lib/variants/*.so; do
  n=$(basename $so .so)
  ECC_B200_LIB=$PWD/$so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "u16 or config4 or hot or lattice or affine" 2>&1 | tail -1 | sed "s/^/$n pytest: /" >> gpurun_out/${TAG}_summary.txt
  ECC_B200_LIB=$PWD/$so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --legs c4 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['legs']['C4']; print('$n C4 ms %.3f golden %s' % (c['ms_per_step'], c['golden_ok']))" >> gpurun_out/${TAG}_summary.txt
done
cat gpurun_out/${TAG}_summary.txt
