#!/bin/bash
# gpu tests + headline benches (cfg2 per ws variant, cfg3, small cholesky)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
for v in 3 4 5; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --variant $v > gpurun_out/bench_v$v.log 2>&1
  echo "cfg2 variant $v: $(grep -o '"value": [0-9.]*' gpurun_out/bench_v$v.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/bench_v$v.log)"
done
timeout 900 bash tools/gpu_cfg3.sh 5 3
timeout 300 python tools/bench_cholesky.py --O 40 --V 200 --tile 40 --nl 480 --ltile 240 --ws-gb 8 > gpurun_out/chol_s.log 2>&1; tail -c 400 gpurun_out/chol_s.log
