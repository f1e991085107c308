#!/bin/bash
# Runs the FP64 peak probes on one B200 with nvidia-smi clock sampling.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/probe_fp64 > gpurun_out/probe_fp64.jsonl 2>&1
python tools/probe_dgemm.py >> gpurun_out/probe_fp64.jsonl 2>&1
kill $SMI
nproc > gpurun_out/probe_host.txt; lscpu | head -20 >> gpurun_out/probe_host.txt
cat gpurun_out/probe_fp64.jsonl
