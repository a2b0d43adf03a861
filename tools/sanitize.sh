#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_driver.py).  Logs under $1 (default
# gpurun_out/sanitize).  Each tool's log ends with its "ERROR SUMMARY".
O=${1:-gpurun_out/sanitize}; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for part in decode prop flash dense bernoulli seqshard host; do
    timeout 900 $CS --tool $tool --error-exitcode 0 --print-limit 50 python tools/sanitize_driver.py $part \
      > $O/${tool}_${part}.log 2>&1
    echo "$tool $part: $(grep -h 'SUMMARY' $O/${tool}_${part}.log | tail -1)" >> $O/summary.txt
  done
done
cat $O/summary.txt
