#!/bin/bash
# GEMM2 (long K) m-block sweep: DRAM bytes and duration per GEMM launch under ncu
# (serialised, cold L2), and the C2 bench step with each setting. Outputs in gpurun_out/gm/.
mkdir -p gpurun_out/gm
for gm in 4 6 8 12 16; do
  AURORA_GEMM_GM_LONGK=$gm timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:grouped_gemm_2sm_kernel -s 4 -c 2 --csv \
    python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/gm/ncu_gm$gm.csv 2>/dev/null
done
for rep in 1 2; do
  for gm in 4 8 12 16; do
    AURORA_GEMM_GM_LONGK=$gm timeout 600 python bench.py --no-cpu-baseline > gpurun_out/gm/bench_gm${gm}_$rep.json 2>/dev/null
  done
done
