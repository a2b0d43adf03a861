#!/bin/bash
O=gpurun_out/${1:-r02_v47}; mkdir -p $O
for i in 1 2; do timeout 120 python tools/c5_prof.py >> $O/c5.json 2>&1; done
timeout 120 python tools/sample_trace.py > $O/trace_c5.json 2>&1
timeout 600 python tools/path_sweep.py 32 256,512 > $O/path_sweep.json 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_extended.py -m gpu -q -x -rf -k "config5 or bernoulli or config3" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
cat $O/c5.json $O/trace_c5.json $O/path_sweep.json; tail -n 3 $O/pytest.log
