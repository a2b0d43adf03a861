#!/bin/bash
O=gpurun_out/${1:-r02_v65}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -rf -k "dense" > $O/pytest_dense.log 2>&1; echo "rc=$?" >> $O/pytest_dense.log
for R in 2 8; do CFG=4 R=$R timeout 120 python tools/sample_trace.py >> $O/trace_c4.json 2>&1; done
tail -n 2 $O/pytest_dense.log; cat $O/trace_c4.json
