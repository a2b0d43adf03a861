#!/bin/bash
# One GPU session: tests, bench, ncu launch list + full captures.  Output under gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-extras > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_stream -s 4 -c 1 -o gpurun_out/prof_score -f \
   python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-extras > gpurun_out/ncu_score.log 2>&1
ls -la gpurun_out
