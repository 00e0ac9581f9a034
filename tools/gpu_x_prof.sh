#!/bin/bash
# full ncu capture (source-level) of the X-only two-group pass-1 kernel on c4
mkdir -p gpurun_out
python tools/prof_eval.py c4 4 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:k_eval_x -s 2 -c 1 -o gpurun_out/eval_x_c4 -f python tools/prof_eval.py c4 3 > gpurun_out/ncu_eval_x.log 2>&1
tail -1 gpurun_out/ncu_eval_x.log
