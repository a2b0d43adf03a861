#!/bin/bash
# Config-5 per-kernel launch list (weights / Bernoulli stream / sampler) under ncu.
O=gpurun_out/${1:-c5}; mkdir -p $O
K=3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
   --log-file $O/c5_launches.csv python tools/c5_prof.py > $O/c5_ncu.log 2>&1
