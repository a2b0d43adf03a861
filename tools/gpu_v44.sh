#!/bin/bash
O=gpurun_out/${1:-r02_v44}; mkdir -p $O
timeout 120 python tools/sample_trace.py > $O/trace_c5.json 2>&1
CFG=3 timeout 120 python tools/sample_trace.py > $O/trace_c3.json 2>&1
CFG=3 S=512 timeout 120 python tools/sample_trace.py > $O/trace_c3_512.json 2>&1
timeout 120 python tools/dense_prof.py > $O/dense.json 2>&1
timeout 120 python tools/dense_prof.py >> $O/dense.json 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -rf -k "dense" > $O/pytest_dense.log 2>&1; echo "rc=$?" >> $O/pytest_dense.log
cat $O/trace_c5.json $O/trace_c3.json $O/trace_c3_512.json $O/dense.json; tail -n 2 $O/pytest_dense.log
