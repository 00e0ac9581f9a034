#!/bin/bash
# Round-2 evidence: ncu launch list of the default bench command, full captures of the Newton-step
# kernels (tile-DAG Cholesky and backward solve at the c4 / c5 n_p), of the c5 pass-1 kernel, and a
# launch list of a c5 Newton fit. Every ncu command runs only after the same command exited 0 without it.
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/prof_bench_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/ncu_launch.log 2>&1
echo "bench launch list rc=$?"
python tools/prof_spd.py 5049,1779 3 > gpurun_out/spd_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_chol_dag|k_trsv_bwd" -c 4 \
    -o gpurun_out/chol_dag_r2 -f python tools/prof_spd.py 5049,1779 1 > gpurun_out/ncu_chol.log 2>&1
echo "chol capture rc=$?"
python tools/prof_eval.py c5 3 > gpurun_out/prof_eval_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_eval_kernel -s 2 -c 1 \
    -o gpurun_out/eval_c5_r2 -f python tools/prof_eval.py c5 3 > gpurun_out/ncu_eval.log 2>&1
echo "eval capture rc=$?"
python tools/prof_hess.py c5 1 fit > gpurun_out/fit_c5_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fit_c5_r2.csv \
    python tools/prof_hess.py c5 1 fit > gpurun_out/ncu_fit_c5.log 2>&1
echo "fit launch list rc=$?"
ls gpurun_out
