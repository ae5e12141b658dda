#!/bin/bash
# compute-sanitizer over the device paths (the driver checks every result
# against the oracle) and over the reference's own chunk-level test programs.
TAG=${1:-san}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_driver.py > gpurun_out/${TAG}_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/${TAG}_${tool}.log
  tail -3 gpurun_out/${TAG}_${tool}.log
done
for t in test_kernel test_value_index test_streaming; do
  timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 tests/cpp/bin/ref_$t > gpurun_out/${TAG}_ref_$t.log 2>&1
  echo "ref_$t memcheck rc=$?" >> gpurun_out/${TAG}_ref_$t.log
  tail -3 gpurun_out/${TAG}_ref_$t.log
done
