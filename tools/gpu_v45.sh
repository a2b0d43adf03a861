#!/bin/bash
O=gpurun_out/${1:-r02_v45}; mkdir -p $O
for i in 1 2; do
SANTA_BERN_NO_KEEPL2=1 timeout 120 python tools/c5_prof.py >> $O/c5_nokeep.json 2>&1
timeout 120 python tools/c5_prof.py >> $O/c5_keep.json 2>&1
done
timeout 120 python tools/sample_trace.py > $O/trace_c5.json 2>&1
SANTA_BERN_NO_KEEPL2=1 timeout 120 python tools/sample_trace.py > $O/trace_c5_nokeep.json 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -rf -k "bernoulli or config5" > $O/pytest_c5.log 2>&1; echo "rc=$?" >> $O/pytest_c5.log
cat $O/c5_nokeep.json $O/c5_keep.json $O/trace_c5.json $O/trace_c5_nokeep.json; tail -n 2 $O/pytest_c5.log
