#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "kernel_paths" > gpurun_out/paths.log 2>&1; tail -2 gpurun_out/paths.log
# Round-1 evidence: bench line, ncu launch list of the same bench command, full captures of the
# dominant kernel (J1 main GEMM, k_pipe_gemm<128>) and of the weight materialisation (k_frag, the per-evaluation weights).
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
cat gpurun_out/bench_r1.json
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/prof_bench_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r1.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/ncu_launch.log 2>&1
python tools/prof_hess.py c4 2 > gpurun_out/prof_hess_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_pipe_gemm -s 0 -c 1 \
    -o gpurun_out/j1_c4_r1 python tools/prof_hess.py c4 1 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:k_frag -s 1 -c 1 \
    -o gpurun_out/afrag_c4_r1 python tools/prof_hess.py c4 1 > gpurun_out/ncu_afrag.log 2>&1
python tools/prof_hess.py c5 2 fit > gpurun_out/fit_c5_r1.log 2>&1
tail -2 gpurun_out/fit_c5_r1.log
