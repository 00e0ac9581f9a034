#!/bin/bash
mkdir -p gpurun_out
python tools/prof_eval.py c5 6 2>&1 | tail -1
MNL_NO_YZW=1 python tools/prof_eval.py c5 6 2>&1 | tail -1
python tools/prof_eval.py c4 6 2>&1 | tail -1
python tools/prof_eval.py c3 6 2>&1 | tail -1
python tools/prof_eval.py c2 6 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_w6.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gputests_w6.log
