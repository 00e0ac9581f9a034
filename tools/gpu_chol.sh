# Cholesky / Newton-step solve: parity tests, event timings, ncu launch list of the solves
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chol or spd or fit_parity or singular or std_errors" > gpurun_out/chol_tests.log 2>&1; tail -3 gpurun_out/chol_tests.log
timeout 300 python tools/prof_spd.py 18,64,189,969,1779,3100,5049 10 2>&1 | tail -8
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_spd.csv \
   python tools/prof_spd.py 18,189,969,1779,5049 3 > gpurun_out/ncu_spd.log 2>&1; echo ncu=$?
python tools/launches.py gpurun_out/launches_spd.csv 2>&1 | tail -30
