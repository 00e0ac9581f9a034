#!/bin/bash
# group-mapping pass 1: c5 timing (new and old path), parity suite
mkdir -p gpurun_out
python tools/prof_eval.py c5 8 2>&1 | tail -1
MNL_NO_YZW=1 python tools/prof_eval.py c5 8 2>&1 | tail -1
python tools/prof_eval.py c1 4 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_w1.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gputests_w1.log
