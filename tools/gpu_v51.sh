#!/bin/bash
O=gpurun_out/${1:-r02_v51}; mkdir -p $O
timeout 300 python -m pytest tests -m gpu -q -x -rf -k "bernoulli or config5 or paged_feature" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 3 $O/pytest.log
for i in 1 2; do timeout 120 python tools/c5_prof.py >> $O/c5.json 2>&1; done
timeout 120 python tools/sample_trace.py > $O/trace_c5.json 2>&1
cat $O/c5.json $O/trace_c5.json
