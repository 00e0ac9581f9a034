mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "std_errors or predict" > gpurun_out/se_tests.log 2>&1; tail -15 gpurun_out/se_tests.log
for c in c3 c5 c4; do python tools/prof_hess.py $c 2 se 2>&1 | tail -1; done
