#!/bin/bash
# full ncu capture (source-level) of the group-mapping pass 1 on c5
mkdir -p gpurun_out
python tools/prof_eval.py c5 4 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:k_eval_w -s 2 -c 1 -o gpurun_out/eval_w_c5 -f python tools/prof_eval.py c5 3 > gpurun_out/ncu_eval_w.log 2>&1
tail -1 gpurun_out/ncu_eval_w.log
