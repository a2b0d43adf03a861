#!/bin/bash
# quick GPU check: gpu tests + bench + launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-extras > gpurun_out/ncu_launch_bench.log 2>&1
