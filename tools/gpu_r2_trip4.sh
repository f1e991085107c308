#!/bin/bash
# 4-GPU box: (T) tests, cost-balanced split at 1/2/4 GPUs, multi-GPU parity
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_triples.py -q -m gpu > gpurun_out/r2g_test.log 2>&1; echo rc=$? >> gpurun_out/r2g_test.log
timeout 600 python tools/bench_triples.py --steps 3 > gpurun_out/r2g_trip_n1.jsonl 2>&1
timeout 600 python tools/bench_triples.py --spin --steps 3 > gpurun_out/r2g_trip_spin_n1.jsonl 2>&1
for N in 2 4; do
  timeout 600 $R --nproc-per-node $N --master-port 2971$N tools/bench_triples.py --steps 3 --cpu-triples 0 > gpurun_out/r2g_trip_n$N.jsonl 2>&1
  timeout 600 $R --nproc-per-node $N --master-port 2972$N tools/bench_triples.py --spin --steps 3 --cpu-triples 0 > gpurun_out/r2g_trip_spin_n$N.jsonl 2>&1
done
for N in 2 4; do timeout 600 $R --nproc-per-node $N --master-port 2973$N tests/mgpu_triples_check.py > gpurun_out/r2g_mgpu_n$N.log 2>&1; echo rc=$? >> gpurun_out/r2g_mgpu_n$N.log; done
tail -2 gpurun_out/r2g_test.log
for f in gpurun_out/r2g_trip*.jsonl; do echo $f; grep -o '"ms_per_step": [0-9.]*\|"energy": [-0-9.e]*\|"alg_tflops": [0-9.]*\|"exec_tflops": [0-9.]*' $f | head -4 | tr '\n' ' '; echo; done
tail -3 gpurun_out/r2g_mgpu_n2.log gpurun_out/r2g_mgpu_n4.log
