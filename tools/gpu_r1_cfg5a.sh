#!/bin/bash
# GPU round: full gpu test suite (incl. 2-GPU checks), small configs[4]-shaped ladders (Bm and two-pass,
# 1 and 2 GPUs) with samples, weak-scaling points at N=1 and N=2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
run() { local n=$1; shift; local tag=$1; shift
  if [ "$n" = 1 ]; then timeout 600 python tools/bench_cfg5.py "$@" > gpurun_out/cfg5_$tag.log 2>&1
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n tools/bench_cfg5.py "$@" > gpurun_out/cfg5_$tag.log 2>&1; fi
  echo rc=$? >> gpurun_out/cfg5_$tag.log; }
run 1 small_n1 --O 24 --V 80 --tile 16 --ltile 50 --ws-gb 0.2 --samples-out gpurun_out/cfg5_samples_small_n1.json
run 2 small_n2_2pass --O 24 --V 80 --tile 16 --ltile 50 --ws-gb 0.01 --samples-out gpurun_out/cfg5_samples_small_n2_2pass.json
run 2 weak_n2 --weak --ws-gb 56 --samples-out gpurun_out/cfg5_samples_weak_n2.json
run 1 weak_n1 --weak --ws-gb 40 --samples-out gpurun_out/cfg5_samples_weak_n1.json
