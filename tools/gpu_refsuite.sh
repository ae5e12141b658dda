#!/bin/bash
# The reference's own tests against the drop-in (built here, run on the box).
TAG=${1:-rs}
mkdir -p gpurun_out
for t in test_streaming test_kernel test_value_index test_curve; do
  timeout 600 tests/cpp/bin/ref_$t > gpurun_out/${TAG}_$t.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_$t.log
  tail -2 gpurun_out/${TAG}_$t.log
done
(cd /tmp && timeout 1200 $GRAFT_REPO_ROOT/tests/cpp/bin/ref_acceptance) > gpurun_out/${TAG}_acceptance.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_acceptance.log
cat gpurun_out/${TAG}_acceptance.log
