#!/bin/bash
# dense_split_kernel variants (libs under gpurun_in/<tag>/, built with -DSANTA_DENSE_*); env B (batch)
O=gpurun_out/${1:-dense_ab}; mkdir -p $O
for i in 1 2; do
  echo -n "B${B:-1} base " >> $O/dense.txt; timeout 300 python tools/dense_prof.py >> $O/dense.txt 2>&1
  for t in $(ls gpurun_in); do
    echo -n "B${B:-1} $t " >> $O/dense.txt; SANTA_LIB_PATH=$PWD/gpurun_in/$t/libsanta.so timeout 300 python tools/dense_prof.py >> $O/dense.txt 2>&1
  done
done
cat $O/dense.txt
