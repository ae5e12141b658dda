#!/bin/bash
# Full GPU suite + the default bench line (C2 + C4/C5 legs + CPU arm).
TAG=${1:-f}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -5 gpurun_out/${TAG}_pytest.log
python - <<PY
import json
d=json.loads(open("gpurun_out/${TAG}_bench.json").read().strip().splitlines()[-1])
print("C2 kernel_ms %.4f frac %.4f value %.1f e2e %.1f" % (d["kernel_ms"], d["roofline"]["frac"], d["value"], d["e2e"]["value"]))
for k,v in d.get("legs",{}).items(): print(k, v.get("ms_per_step"), v.get("golden_ok"), v.get("value"))
print("cpu", d.get("cpu_baseline"))
PY
