mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "yz_paths or shapes or hessvec or c5 or c1 or c2 or random" > gpurun_out/eval_tests.log 2>&1; tail -2 gpurun_out/eval_tests.log
python tools/prof_eval.py c5 8 2>&1 | tail -1
python tools/prof_eval.py c4 8 2>&1 | tail -1
python tools/prof_hess.py c5 2 fit 2>&1 | tail -1
