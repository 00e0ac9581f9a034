# Hessian-path changes: parity subset (every kernel path, ragged shapes, full-size c5, fits) + timings
mkdir -p gpurun_out
python tools/time_hess.py c2 c3 c5 2>&1 | grep -v Warn | tail -6
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dp.py -x -q -k "kernel_paths or full_hessian or shapes or fit_parity or full_size and c5 or small or dp_" > gpurun_out/hess_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/hess_tests.log
