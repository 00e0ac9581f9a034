#!/bin/bash
# Step 0: measure FP64 DMMA/DFMA throughput and the box's host.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/step0_clocks.csv &
SMI=$!
./tools/fp64_peak > gpurun_out/fp64_peak.json 2> gpurun_out/fp64_peak.err
kill $SMI
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|Socket|Thread|Core" >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
nvidia-smi >> gpurun_out/host.txt
cat gpurun_out/fp64_peak.json
