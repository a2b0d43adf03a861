#!/bin/bash
O=gpurun_out/${1:-r02_v71}; mkdir -p $O
for B in 1 32; do for v in pdl nopdl; do
  if [ $v = nopdl ]; then export SANTA_SCORE_NO_PDL=1; else unset SANTA_SCORE_NO_PDL; fi
  echo -n "B$B $v " >> $O/ab.txt; B=$B timeout 200 python tools/score_prof.py >> $O/ab.txt 2>&1
done; done
unset SANTA_SCORE_NO_PDL
timeout 600 python tools/path_sweep.py 32 128,256 > $O/sweep_pdl.json 2>&1
SANTA_SCORE_NO_PDL=1 timeout 600 python tools/path_sweep.py 32 128,256 > $O/sweep_nopdl.json 2>&1
cat $O/ab.txt $O/sweep_pdl.json $O/sweep_nopdl.json
