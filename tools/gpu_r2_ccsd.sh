#!/bin/bash
# round 2: textbook CCSD iteration -- tests, then configs[3] at N GPUs
mkdir -p gpurun_out
N=${1:-1}
timeout 600 python -m pytest tests/test_ccsd_iteration.py -q -m gpu -x > gpurun_out/r2c_test.log 2>&1; echo rc=$? >> gpurun_out/r2c_test.log
nvidia-smi --query-gpu=memory.total,clocks.sm --format=csv > gpurun_out/r2c_smi.txt
if [ "$N" == "1" ]; then
  timeout 1500 python tools/bench_ccsd.py --steps 1 --warmup 2 > gpurun_out/r2c_bench_n1.jsonl 2> gpurun_out/r2c_bench_n1.err
else
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 tools/bench_ccsd.py --steps 1 --warmup 2 > gpurun_out/r2c_bench_n$N.jsonl 2> gpurun_out/r2c_bench_n$N.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29556 tests/mgpu_ccsd_check.py > gpurun_out/r2c_mgpu_n$N.log 2>&1
fi
tail -3 gpurun_out/r2c_test.log; tail -c 3000 gpurun_out/r2c_bench_n$N.jsonl; tail -5 gpurun_out/r2c_bench_n$N.err
