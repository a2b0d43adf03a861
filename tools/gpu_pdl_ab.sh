#!/bin/bash
O=gpurun_out/${1:-pdl_ab}; mkdir -p $O
for i in 1 2; do
  echo -n "base " >> $O/ab.txt; timeout 200 python tools/score_prof.py >> $O/ab.txt 2>&1
  echo -n "pdl  " >> $O/ab.txt; SANTA_LIB_PATH=$PWD/gpurun_in/pdl/libsanta.so timeout 200 python tools/score_prof.py >> $O/ab.txt 2>&1
done
SANTA_LIB_PATH=$PWD/gpurun_in/pdl/libsanta.so timeout 900 python -m pytest tests -m gpu -q -x -rf -k "parity or decode_loop or fullsize" > $O/pytest_pdl.log 2>&1; echo "pdl tests rc=$?" >> $O/ab.txt
cat $O/ab.txt; tail -n 2 $O/pytest_pdl.log
