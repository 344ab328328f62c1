#!/bin/bash
# Round-2 ncu evidence (gpurun_out/r02p/): launch lists of our kernels only (C2, C5) and one
# --set full capture of the router, pack, dispatch engine and aggregate (C2) and the C5 E > n kernels.
mkdir -p gpurun_out/r02p
K='regex:route|pack|schedule|engine|gemm|aggregate|combine|expert|hist|gather|prepare'
for c in c2 c5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 200 --csv \
    --log-file gpurun_out/r02p/launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline \
    > /dev/null 2>&1
done
for k in route_tma_kernel pack_kernel engine_tma_kernel aggregate_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/r02p/$k \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
for k in route_units_kernel route_tail_kernel expert_reduce_kernel engine_tma_kernel pack_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/r02p/c5_$k \
    python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
python tools/ncu_summary.py gpurun_out/r02p/ncu_c2.json gpurun_out/r02p/route_tma_kernel.ncu-rep \
  gpurun_out/r02p/pack_kernel.ncu-rep gpurun_out/r02p/engine_tma_kernel.ncu-rep gpurun_out/r02p/aggregate_kernel.ncu-rep
python tools/ncu_summary.py gpurun_out/r02p/ncu_c5.json gpurun_out/r02p/c5_*.ncu-rep
ls -la gpurun_out/r02p
