#!/bin/bash
O=gpurun_out/${1:-r02_v46}; mkdir -p $O
for i in 1 2; do timeout 120 python tools/c5_prof.py >> $O/c5.json 2>&1; done
timeout 120 python tools/sample_trace.py > $O/trace_c5.json 2>&1
CFG=3 timeout 120 python tools/sample_trace.py > $O/trace_c3.json 2>&1
timeout 600 python tools/path_sweep.py 16,32 64,256,512 > $O/path_sweep.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
cat $O/c5.json $O/trace_c5.json $O/trace_c3.json $O/path_sweep.json; tail -n 3 $O/pytest_gpu.log
