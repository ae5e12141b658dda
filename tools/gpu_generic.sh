#!/bin/bash
# Generic (tournament) kernels: timing probe + the full GPU suite.
TAG=${1:-g}
mkdir -p gpurun_out
timeout 300 python tools/probe_generic.py > gpurun_out/${TAG}_probe.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
cat gpurun_out/${TAG}_probe.jsonl; tail -15 gpurun_out/${TAG}_pytest.log
