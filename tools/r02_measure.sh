#!/bin/bash
# On the GPU box: the C2 bench line, the bench's multi-process test, the launch list of
# one step and ncu --set full captures of the expert GEMMs and K2. Outputs in gpurun_out/r02/.
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02/smi.txt
timeout 900 python bench.py > gpurun_out/r02/bench_c2.json 2> gpurun_out/r02/bench_c2.err
timeout 900 python -m pytest tests/test_bench_gpu.py -q > gpurun_out/r02/test_bench_gpu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/r02/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:grouped_gemm_2sm_kernel -s 2 -c 2 \
  -o gpurun_out/r02/gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02/gemm.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:aurora_schedule_kernel -s 2 -c 1 \
  -o gpurun_out/r02/k2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02/k2.log 2>&1
python tools/ncu_summary.py gpurun_out/r02/ncu_gemm.json gpurun_out/r02/gemm.ncu-rep > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02/ncu_k2.json gpurun_out/r02/k2.ncu-rep > /dev/null 2>&1
ls -la gpurun_out/r02
