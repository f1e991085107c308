#!/bin/bash
# GPU tests + bench of every contraction kernel variant on cfg2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
for v in "$@"; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --variant $v > gpurun_out/bench_v$v.log 2>&1
  echo "variant $v: $(grep -o '"value": [0-9.]*' gpurun_out/bench_v$v.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/bench_v$v.log)"
done
tail -n 4 gpurun_out/pytest_gpu.log
