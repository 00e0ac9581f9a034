#!/bin/bash
# Round-2 final evidence: full GPU suite + smoke, default bench line, ncu launch list of the same
# bench command, one full capture of the J1 main GEMM (traffic) on c4, per-config table.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_final.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"; cat gpurun_out/bench_final.json
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/prof_bench_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r2_final.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
python tools/prof_hess.py c4 2 > gpurun_out/prof_hess_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_pipe_gemm -s 0 -c 1 \
    -o gpurun_out/j1_c4_r2 -f python tools/prof_hess.py c4 1 > gpurun_out/ncu_j1.log 2>&1; echo "j1 capture rc=$?"
timeout 900 python tools/config_table.py > gpurun_out/config_table_r2.json 2> gpurun_out/config_table.err; echo "config table rc=$?"
