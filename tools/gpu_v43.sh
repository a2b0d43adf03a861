#!/bin/bash
O=gpurun_out/${1:-r02_v43}; mkdir -p $O
for i in 1 2; do
SANTA_SAMPLE_MINB=1 timeout 120 python tools/c5_prof.py >> $O/c5_minb1.json 2>&1
timeout 120 python tools/c5_prof.py >> $O/c5_auto.json 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python tools/path_sweep.py 4,8,16,32 256,512 > $O/path_sweep.json 2>&1
K=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sample_gather -s 1 -c 1 -o $O/prof_c5_sample -f \
   python tools/c5_prof.py > $O/ncu_c5_sample.log 2>&1
cat $O/c5_minb1.json $O/c5_auto.json; tail -n 3 $O/pytest_gpu.log
