mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chol or fit_parity or singular or std_errors" > gpurun_out/chol_tests.log 2>&1; tail -3 gpurun_out/chol_tests.log
for n in 5049 3500 1779 969; do python tools/prof_chol.py $n 3 2>&1 | tail -1; done
for n in 5049 1779; do MNL_CHOL_STREAMS=1 python tools/prof_chol.py $n 3 2>&1 | tail -1; done
