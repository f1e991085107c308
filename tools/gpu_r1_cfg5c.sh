#!/bin/bash
# 2 GPUs: gpu tests (incl. 2-GPU checks), configs[4] ladder small (samples), weak N=1/N=2, strong N=2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
run() { local n=$1; shift; local tag=$1; shift
  if [ "$n" = 1 ]; then timeout 900 python tools/bench_cfg5.py "$@" > gpurun_out/cfg5_$tag.log 2>&1
  else timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n tools/bench_cfg5.py "$@" > gpurun_out/cfg5_$tag.log 2>&1; fi
  echo rc=$? >> gpurun_out/cfg5_$tag.log; }
run 2 small_n2 --O 24 --V 80 --tile 16 --ltile 50 --samples-out gpurun_out/cfg5_samples_small_n2.json
# run 1 weak_n1 --weak --samples-out gpurun_out/cfg5_samples_weak_n1.json
run 2 weak_n2 --weak --samples-out gpurun_out/cfg5_samples_weak_n2.json
run 2 strong_n2 --samples-out gpurun_out/cfg5_samples_strong_n2.json
