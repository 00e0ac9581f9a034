# c5 pass 1: event timing, one full ncu capture (source-level) of the gradient pass
mkdir -p gpurun_out
python tools/prof_eval.py c5 8 2>&1 | tail -1
python tools/prof_eval.py c4 8 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:k_eval_kernel -s 2 -c 1 -o gpurun_out/eval_c5_r2 -f python tools/prof_eval.py c5 3 > gpurun_out/ncu_eval_c5.log 2>&1
tail -1 gpurun_out/ncu_eval_c5.log
