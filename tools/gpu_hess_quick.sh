mkdir -p gpurun_out
python tools/prof_hess.py c4 3 eval 2>&1 | tail -1
python tools/prof_hess.py c5 3 eval 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "kernel_paths or full_hessian or shapes or fit_parity or full_size" > gpurun_out/hess_tests.log 2>&1; tail -3 gpurun_out/hess_tests.log
