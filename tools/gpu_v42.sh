#!/bin/bash
O=gpurun_out/${1:-r02_v42}; mkdir -p $O
for i in 1 2; do
SANTA_SAMPLE_MINB=1 timeout 120 python tools/c5_prof.py >> $O/c5_minb1.json 2>&1
timeout 120 python tools/c5_prof.py >> $O/c5_auto.json 2>&1
done
timeout 900 python -m pytest tests/test_gpu_peer.py -m gpu -q -x -rf -s > $O/pytest_peer.log 2>&1; echo "rc=$?" >> $O/pytest_peer.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_extended.py -m gpu -q -x -rf -s -k "config5 or bernoulli" > $O/pytest_c5.log 2>&1; echo "rc=$?" >> $O/pytest_c5.log
K=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sample_gather -s 1 -c 1 -o $O/prof_c5_sample -f \
   python tools/c5_prof.py > $O/ncu_c5_sample.log 2>&1
cat $O/c5_minb1.json $O/c5_auto.json; tail -3 $O/pytest_peer.log $O/pytest_c5.log
