#!/bin/bash
# Session baseline: GPU suite, smoke, bench line, config table.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_s4.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_s4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s4.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_s4.log
timeout 900 python bench.py > gpurun_out/bench_s4.json 2> gpurun_out/bench_s4.err; echo "bench rc=$?"; cat gpurun_out/bench_s4.json
timeout 900 python tools/config_table.py > gpurun_out/config_table_s4.json 2> gpurun_out/config_table_s4.err; echo "config table rc=$?"
