#!/bin/bash
mkdir -p gpurun_out
python tools/prof_eval.py c5 6 2>&1 | tail -1
python tools/prof_eval.py c1 4 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "team_mapping or yz_paths or nonfinite or full_size or golden-c5 or hessvec or fit_parity_small" > gpurun_out/gputests_w4.log 2>&1; echo "tests rc=$?"; tail -12 gpurun_out/gputests_w4.log
