#!/bin/bash
mkdir -p gpurun_out
MNL_W_NBW=2 python tools/prof_eval.py c5 6 2>&1 | tail -1
MNL_W_NBW=1 python tools/prof_eval.py c5 6 2>&1 | tail -1
python tools/dbg_nan.py 2>&1 | head -3
MNL_W_NBW=2 ncu --set full --clock-control none --import-source on -k regex:k_eval_w -s 2 -c 1 -o gpurun_out/eval_w_c5 -f python tools/prof_eval.py c5 3 > gpurun_out/ncu_eval_w.log 2>&1
tail -1 gpurun_out/ncu_eval_w.log
