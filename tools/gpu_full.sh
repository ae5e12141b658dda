#!/bin/bash
# Full evidence pass (under gpurun): tests, bench lines (both arms), launch
# list + full ncu capture of the bench kernel, per-config numbers and full
# captures of the other configs' kernels.  Usage: bash tools/gpu_full.sh TAG
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $OUT/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/${TAG}_bench_reference_arm.json 2>> $OUT/${TAG}_bench.err
timeout 600 python tools/bench_configs.py C1 C3 C4 > $OUT/${TAG}_configs.jsonl 2>> $OUT/${TAG}_bench.err
timeout 300 python tools/probe_2d.py > $OUT/${TAG}_probe_2d.txt 2>&1
timeout 300 python tools/probe_f32.py > $OUT/${TAG}_probe_f32.txt 2>&1
timeout 300 python tools/probe_smooth.py > $OUT/${TAG}_probe_smooth.txt 2>&1
timeout 600 python tools/probe_e2e_dense.py > $OUT/${TAG}_probe_e2e_dense.txt 2>&1
timeout 300 python tools/bench_pipeline.py 512 5 128 > $OUT/${TAG}_pipeline.jsonl 2>&1
timeout 300 ./tests/cpp/bin/e2e_c > $OUT/${TAG}_e2e_c_abi.jsonl 2>&1
timeout 600 python tools/c5_sharded.py --side 2048 > $OUT/${TAG}_c5_2048.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/${TAG}_launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_u8_3d -s 2 -c 1 -o $OUT/${TAG}_k_u8_3d \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_c34_launches.csv \
   python tools/bench_configs.py C3 C4 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch16 -s 2 -c 1 -o $OUT/${TAG}_k_batch16 \
   python tools/bench_configs.py C3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_u16_3d|k_affine_keys" -s 2 -c 2 -o $OUT/${TAG}_k_u16_3d \
   python tools/bench_configs.py C4 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_u8_2d|k_u16_2d" -s 2 -c 2 -o $OUT/${TAG}_k_2d \
   python tools/probe_2d.py > /dev/null 2>&1
echo done
