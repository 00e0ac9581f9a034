mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "yz_paths or shapes or hessvec or c5 or c1" > gpurun_out/yzs_tests.log 2>&1; tail -5 gpurun_out/yzs_tests.log
for c in c1 c5; do python tools/prof_eval.py $c 8 2>&1 | tail -1; done
python tools/prof_hess.py c5 2 fitcg 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:k_eval_kernel -s 2 -c 1 -o gpurun_out/eval_c5_yzs9 python tools/prof_eval.py c5 3 > gpurun_out/ncu_eval_c5.log 2>&1
tail -1 gpurun_out/ncu_eval_c5.log
