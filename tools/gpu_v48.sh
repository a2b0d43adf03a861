#!/bin/bash
O=gpurun_out/${1:-r02_v48}; mkdir -p $O
for i in 1 2; do for v in 4 5 6 1; do echo -n "v$v " >> $O/c5.txt; SANTA_SAMPLE_MINB=$v timeout 120 python tools/c5_prof.py >> $O/c5.txt 2>&1; done; done
cat $O/c5.txt
