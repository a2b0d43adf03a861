#!/bin/bash
O=gpurun_out/${1:-score_ab}; mkdir -p $O
for B in 1 32; do
  echo -n "B$B base " >> $O/score.txt; B=$B timeout 200 python tools/score_prof.py >> $O/score.txt 2>&1
  for t in $(ls gpurun_in); do
    echo -n "B$B $t " >> $O/score.txt; B=$B SANTA_LIB_PATH=$PWD/gpurun_in/$t/libsanta.so timeout 200 python tools/score_prof.py >> $O/score.txt 2>&1
  done
done
cat $O/score.txt
