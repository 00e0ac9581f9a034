#!/bin/bash
# Round-1 (second session) evidence: full GPU suite, bench line, ncu launch list of the bench
# command, full capture of the YZS pass-1 kernel on c5, launch list of a c5 Newton fit.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; cat gpurun_out/bench_r1b.json; tail -2 gpurun_out/bench_r1b.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/prof_bench_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r1b.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/ncu_launch.log 2>&1
python tools/prof_eval.py c5 3 > gpurun_out/prof_eval_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_eval_kernel -s 2 -c 1 \
    -o gpurun_out/eval_c5_r1b python tools/prof_eval.py c5 3 > gpurun_out/ncu_eval.log 2>&1
python tools/prof_hess.py c5 1 fit > gpurun_out/fit_c5_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fit_c5_r1b.csv \
    python tools/prof_hess.py c5 1 fit > gpurun_out/ncu_fit_c5.log 2>&1
ls gpurun_out
