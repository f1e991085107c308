#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
for tma in 1 0; do for v in 5 3; do
  TT_TMA=$tma timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --variant $v > gpurun_out/bench_t${tma}_v$v.log 2>&1
  echo "cfg2 tma=$tma variant $v: $(grep -o '"value": [0-9.]*' gpurun_out/bench_t${tma}_v$v.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/bench_t${tma}_v$v.log)"
done; done
TT_TMA=1 timeout 900 bash tools/gpu_cfg3.sh 5
