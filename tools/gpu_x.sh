mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "shapes or full_hessian or c4 or hessvec or kernel_paths" > gpurun_out/x_tests.log 2>&1; tail -3 gpurun_out/x_tests.log
for c in c2 c3 c4; do python tools/prof_eval.py $c 8 2>&1 | tail -1; done
python tools/prof_hess.py c4 3 hv 2>&1 | tail -1
python tools/prof_hess.py c4 1 fitcg 2>&1 | tail -1
