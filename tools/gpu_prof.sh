#!/bin/bash
# full ncu captures of the score and sample kernels (one launch each, after warm-up)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_stream -s 6 -c 1 -o gpurun_out/prof_score -f \
   python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-extras > gpurun_out/ncu_score.log 2>&1
timeout 600 ncu --set full --clock-control none --cache-control none --warp-sampling-interval 0 --import-source on -k regex:sample_gather -s 6 -c 1 -o gpurun_out/prof_sample -f \
   python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-extras > gpurun_out/ncu_sample.log 2>&1
