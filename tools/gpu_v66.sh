#!/bin/bash
O=gpurun_out/${1:-r02_v66}; mkdir -p $O
for R in 2 8; do CFG=4 R=$R timeout 120 python tools/sample_trace.py >> $O/trace_c4.json 2>&1; done
for i in 1 2; do timeout 120 python tools/c5_prof.py >> $O/c5.json 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
python - <<'PY'
import json
for l in open("gpurun_out/r02_v66/trace_c4.json"):
    d = json.loads(l); print({k: v["rel_med_us"] for k, v in d.items() if k.startswith("phase")})
PY
cat $O/c5.json; tail -n 2 $O/pytest_gpu.log
