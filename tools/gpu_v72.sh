#!/bin/bash
O=gpurun_out/${1:-r02_v72}; mkdir -p $O
for B in 1 32; do
  echo -n "B$B cur-pdl " >> $O/ab.txt; B=$B timeout 200 python tools/score_prof.py >> $O/ab.txt 2>&1
  echo -n "B$B cur-nopdl " >> $O/ab.txt; SANTA_SCORE_NO_PDL=1 B=$B timeout 200 python tools/score_prof.py >> $O/ab.txt 2>&1
  echo -n "B$B nowait-nopdl " >> $O/ab.txt; SANTA_SCORE_NO_PDL=1 SANTA_LIB_PATH=$PWD/gpurun_in/nowait/libsanta.so B=$B timeout 200 python tools/score_prof.py >> $O/ab.txt 2>&1
done
cat $O/ab.txt
