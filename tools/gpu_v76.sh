#!/bin/bash
O=gpurun_out/${1:-r02_v76}; mkdir -p $O
for i in 1 2 3; do
  echo -n "one " >> $O/ab.txt; timeout 200 python tools/c5_prof.py >> $O/ab.txt 2>&1
  echo -n "all " >> $O/ab.txt; SANTA_LIB_PATH=$PWD/gpurun_in/btall/libsanta.so timeout 200 python tools/c5_prof.py >> $O/ab.txt 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -x -rf -k "bernoulli or config5 or paged_feature" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/ab.txt
cat $O/ab.txt; tail -n 1 $O/pytest.log
