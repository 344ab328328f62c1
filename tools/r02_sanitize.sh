#!/bin/bash
# compute-sanitizer over the small layer forwards (tools/sanitize_layer.py); summaries in gpurun_out/r02/
mkdir -p gpurun_out/r02
for t in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_layer.py \
    > gpurun_out/r02/sanitize_$t.log 2>&1
  echo "$t exit $?" >> gpurun_out/r02/sanitize_$t.log
done
tail -5 gpurun_out/r02/sanitize_*.log
