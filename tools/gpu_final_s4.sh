#!/bin/bash
# Round-2 (last session) evidence: GPU suite + smoke, default bench line, ncu launch list of the same
# bench command, c5 fit launch list, full captures of the c5 pass-1 kernel (team mapping) and of the c4
# X-only pass-1 kernel, per-config table. Every ncu command runs only after the same command
# exited 0 without it.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_final.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"; cat gpurun_out/bench_final.json
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/prof_bench_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/ncu_launch.log 2>&1; echo "bench launch list rc=$?"
python tools/prof_hess.py c5 1 fit > gpurun_out/fit_c5_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fit_c5_r2.csv \
    python tools/prof_hess.py c5 1 fit > gpurun_out/ncu_fit_c5.log 2>&1; echo "fit launch list rc=$?"
python tools/prof_eval.py c5 3 > gpurun_out/prof_eval_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_eval_w -s 2 -c 1 \
    -o gpurun_out/eval_c5_team_r2 -f python tools/prof_eval.py c5 3 > gpurun_out/ncu_eval.log 2>&1; echo "c5 eval capture rc=$?"
python tools/prof_eval.py c4 3 > gpurun_out/prof_eval4_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_eval_x -s 2 -c 1 \
    -o gpurun_out/eval_c4_xonly_r2 -f python tools/prof_eval.py c4 3 > gpurun_out/ncu_eval4.log 2>&1; echo "c4 eval capture rc=$?"
timeout 900 python tools/config_table.py > gpurun_out/config_table_r2.json 2> gpurun_out/config_table.err; echo "config table rc=$?"
bash tools/gpu_pass1_team_vs_yzs.sh > gpurun_out/team_vs_yzs.log 2>&1; cat gpurun_out/team_vs_yzs.log
