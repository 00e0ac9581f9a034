#!/bin/bash
# round-1 profiling call: launch list of the bench command + one full capture of the J1 DMMA kernel
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_bench_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
python tools/prof_hess.py c4 2 > gpurun_out/prof_hess_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_gen_gemm -s 1 -c 1 \
    -o gpurun_out/prof_c4_gemm python tools/prof_hess.py c4 2 > gpurun_out/ncu_full.log 2>&1
python tools/prof_hess.py c5 2 > gpurun_out/prof_hess_c5.log 2>&1
python tools/prof_hess.py c5 1 fit >> gpurun_out/prof_hess_c5.log 2>&1
tail -3 gpurun_out/ncu_launch.log gpurun_out/ncu_full.log gpurun_out/prof_hess_c5.log
