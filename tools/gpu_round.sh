#!/bin/bash
# One GPU call: gpu tests, smoke, bench, launch list and a full ncu capture of the contraction kernel.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
(timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log)
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$? >> gpurun_out/bench.log
if [ "$1" == "ncu" ]; then
  timeout 300 $B > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
  timeout 300 $B > gpurun_out/plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tt_contract -s 3 -c 1 -o gpurun_out/prof_contract $B > gpurun_out/ncu_full.log 2>&1
  echo ncu_rc=$? >> gpurun_out/ncu_full.log
fi
tail -n 3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log; tail -c 1500 gpurun_out/bench.log
