# small-problem checks: the one-launch Hessian's parity tests (both paths), DP tests, smoke, timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dp.py -x -q -k "small or dp_ or fit_parity_small or ftol or std_errors or random_shapes or nonfinite" > gpurun_out/small_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/small_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python tools/time_hess.py c1 c2 2>&1 | tail -4
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1_fit.csv python tools/prof_hess.py c1 1 fit > gpurun_out/ncu_c1.log 2>&1; echo ncu rc=$?
