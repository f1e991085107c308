#!/bin/bash
# bench.py under torchrun at N GPUs (the driver's scaling run) + the multi-GPU parity scripts
mkdir -p gpurun_out
N=${1:-2}
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N > gpurun_out/r2s_bench_n$N.log 2>&1; echo bench_rc=$? >> gpurun_out/r2s_bench_n$N.log
timeout 1200 python -m pytest tests/test_multigpu.py -q -m gpu > gpurun_out/r2s_mgpu_n$N.log 2>&1; echo rc=$? >> gpurun_out/r2s_mgpu_n$N.log
grep '^{' gpurun_out/r2s_bench_n$N.log | tail -c 1500; tail -3 gpurun_out/r2s_bench_n$N.log; tail -3 gpurun_out/r2s_mgpu_n$N.log
