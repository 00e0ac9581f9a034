mkdir -p gpurun_out
for c in c2 c3 c4 c5; do python tools/prof_eval.py $c 8 2>&1 | tail -1; done > gpurun_out/eval_times.log
cat gpurun_out/eval_times.log
for c in c4 c5; do python tools/prof_hess.py $c 3 hv 2>&1 | tail -1; python tools/prof_hess.py $c 2 fitcg 2>&1 | tail -1; done > gpurun_out/cg.log 2>&1
cat gpurun_out/cg.log
ncu --set full --clock-control none --import-source on -k regex:k_eval_kernel -s 2 -c 1 -o gpurun_out/eval_c5 python tools/prof_eval.py c5 3 > gpurun_out/ncu_eval_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_eval_kernel -s 2 -c 1 -o gpurun_out/eval_c3 python tools/prof_eval.py c3 3 > gpurun_out/ncu_eval_c3.log 2>&1
tail -2 gpurun_out/ncu_eval_c5.log
