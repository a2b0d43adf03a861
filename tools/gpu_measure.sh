#!/bin/bash
# Round-2 end-of-work measurement: tests, smoke, bench (ours + reference arm), ncu launch list and
# --set full captures of the two kernels of the AUTO config-2 step.  Output under gpurun_out/$1.
O=gpurun_out/${1:-measure}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
   --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_stream -s 6 -c 1 -o $O/prof_score -f \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $O/ncu_score.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sample_fast -s 6 -c 1 -o $O/prof_sample -f \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $O/ncu_sample.log 2>&1
ls -la $O
