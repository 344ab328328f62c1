#!/bin/bash
# End-of-round evidence (gpurun_out/final/): GPU tests + smoke, every bench config, the reference arm,
# the C2 / C5 launch lists, one ncu --set full capture of both GEMM launches and of K2, the K2 N = 8
# projection, an 800-config stress run and the tensor-core router's A/B and bound checks.
mkdir -p gpurun_out/final
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/final/gputest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
for c in c2 c3 c3h c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
K='regex:route|pack|schedule|engine|gemm|aggregate|combine|expert|hist|gather|prepare'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 200 --csv \
  --log-file gpurun_out/final/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:grouped_gemm_2sm_kernel -s 2 -c 2 \
  -o gpurun_out/final/gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/final/ncu_gemm.json gpurun_out/final/gemm.ncu-rep > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 200 --csv \
  --log-file gpurun_out/final/launches_c5.csv python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline \
  > /dev/null 2>&1
# K2 as it runs in the C2 layer (cold, serialised) and its schedule-vs-NVLink-need projection
timeout 600 ncu --set full --import-source on --clock-control none -k regex:aurora_schedule -s 2 -c 1 \
  -o gpurun_out/final/k2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/final/ncu_k2.json gpurun_out/final/k2.ncu-rep > /dev/null 2>&1
timeout 900 python tools/k2_n8_projection.py gpurun_out/final/k2_n8_projection.json > /dev/null 2>&1
timeout 900 python tools/stress.py 800 23 > gpurun_out/final/stress.txt 2>&1
# the tensor-core router (E > 8): A/B against the FMA router and its certificate bound on real inputs
for s in 0 1 2; do timeout 300 python tools/route_tc_time.py $s; done > gpurun_out/final/route_tc_time.txt 2>&1
timeout 600 python tools/route_tc_bound.py 2048 > gpurun_out/final/route_tc_bound.txt 2>&1
tail -2 gpurun_out/final/gputest.log; tail -1 gpurun_out/final/smoke.log
