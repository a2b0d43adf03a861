#!/bin/bash
# peer-exchange tests + ncu --set full of the config-5 sampler and the config-2 dense kernel
O=gpurun_out/${1:-r02_v41}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_peer.py -m gpu -q -x -rf -s > $O/pytest_peer.log 2>&1; echo "rc=$?" >> $O/pytest_peer.log
K=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sample_gather -s 1 -c 1 -o $O/prof_c5_sample -f \
   python tools/c5_prof.py > $O/ncu_c5_sample.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_split_kernel -s 3 -c 1 -o $O/prof_dense -f \
   python tools/dense_prof.py > $O/ncu_dense.log 2>&1
ls -la $O
