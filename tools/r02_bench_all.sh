#!/bin/bash
# Round-2 bench lines for every config + the reference arm + the C2 launch list (gpurun_out/r02b/)
mkdir -p gpurun_out/r02b
for c in c2 c3 c3h c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/r02b/bench_$c.json 2> gpurun_out/r02b/bench_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/r02b/bench_reference.json 2> gpurun_out/r02b/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02b/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02b/launches_c5.csv python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline \
  > /dev/null 2>&1
ls -la gpurun_out/r02b
