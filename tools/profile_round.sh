#!/bin/bash
# On the GPU box: launch list of one bench step + one --set full capture of
# each Aurora kernel (C2; C5 for the E > n kernels). Outputs under gpurun_out/prof/.
set -x
mkdir -p gpurun_out/prof
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/prof/bench_under_ncu.log 2>&1
for k in aurora_schedule_kernel engine_tma_kernel route_tma_kernel pack_kernel aggregate_kernel combine_wait_kernel; do
  ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/prof/$k \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof/$k.log 2>&1
done
# both expert GEMM launches of one step (GEMM2 with the combine fused into its epilogue)
ncu --set full --import-source on --clock-control none -k regex:grouped_gemm_2sm_kernel -s 2 -c 2 \
  -o gpurun_out/prof/grouped_gemm_2sm_kernel python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  > gpurun_out/prof/grouped_gemm_2sm_kernel.log 2>&1
# C5 (E > n): balanced router units + top-k tail, row gather, pre-reduction with the fused combine
for k in route_units_kernel route_tail_kernel gather_rows_kernel expert_reduce_kernel; do
  ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/prof/c5_$k \
    python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof/c5_$k.log 2>&1
done
ls -la gpurun_out/prof
