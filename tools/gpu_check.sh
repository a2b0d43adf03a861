#!/bin/bash
# GPU check of the working tree: gpu tests, smoke, bench (default), launch list.  Output under gpurun_out/$TAG.
TAG=${1:-check}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $O/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q -x -rA > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches.csv \
   python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras > $O/ncu_launch_bench.log 2>&1
ls -la $O
