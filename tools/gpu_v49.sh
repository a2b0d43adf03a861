#!/bin/bash
O=gpurun_out/${1:-r02_v49}; mkdir -p $O
for i in 1 2; do timeout 120 python tools/c5_prof.py >> $O/c5.json 2>&1; done
timeout 900 python tools/path_sweep.py 4,8,16,32 64,256,512 > $O/path_sweep.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
cat $O/c5.json $O/path_sweep.json; tail -n 3 $O/pytest_gpu.log
