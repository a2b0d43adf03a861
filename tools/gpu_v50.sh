#!/bin/bash
O=gpurun_out/${1:-r02_v50}; mkdir -p $O
for i in 1 2; do timeout 120 python tools/c5_prof.py >> $O/c5.json 2>&1; done
timeout 600 python -m pytest tests -m gpu -q -x -rf -k "bernoulli or config5" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/gpu_c5_launches.sh r02_v50
cat $O/c5.json; tail -n 2 $O/pytest.log
