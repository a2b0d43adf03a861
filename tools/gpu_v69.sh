#!/bin/bash
O=gpurun_out/${1:-r02_v69}; mkdir -p $O
for i in 1 2; do timeout 120 python tools/dense_prof.py >> $O/dense.json 2>&1; done
B=32 K=20 timeout 300 python tools/dense_prof.py >> $O/dense.json 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -rf -k "dense" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
cat $O/dense.json; tail -n 2 $O/pytest.log
