mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python tools/prof_eval.py c5 8 2>&1 | tail -1
python tools/prof_hess.py c5 2 fit 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fit_c5_q.csv python tools/prof_hess.py c5 1 fit > /dev/null 2>&1; python tools/launches.py gpurun_out/launches_fit_c5_q.csv | grep finalize
