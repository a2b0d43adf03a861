#!/bin/bash
O=gpurun_out/${1:-r02_v68}; mkdir -p $O
for i in 1 2; do timeout 120 python tools/c5_prof.py >> $O/c5.json 2>&1; timeout 200 python tools/score_prof.py >> $O/score.json 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
cat $O/c5.json $O/score.json; tail -n 2 $O/pytest_gpu.log
