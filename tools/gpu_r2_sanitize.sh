#!/bin/bash
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python tools/sanitize_mini.py > gpurun_out/r2s_plain.log 2>&1; echo rc=$? >> gpurun_out/r2s_plain.log
for tool in racecheck synccheck memcheck; do
  timeout 1200 $CS --tool $tool --print-limit 20 python tools/sanitize_mini.py > gpurun_out/r2s_$tool.log 2>&1
  echo rc=$? >> gpurun_out/r2s_$tool.log
done
tail -4 gpurun_out/r2s_*.log
