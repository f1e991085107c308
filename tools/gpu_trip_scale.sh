#!/bin/bash
# (T) energy at O=40 V=200 on 1, 2 and 4 GPUs of one box (strong scaling; energies must agree)
mkdir -p gpurun_out
for n in 1 2 4; do
  if [ $n == 1 ]; then timeout 600 python tools/bench_triples.py > gpurun_out/trip_n$n.log 2>&1
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29531 tools/bench_triples.py > gpurun_out/trip_n$n.log 2>&1; fi
  echo "n=$n rc=$?" >> gpurun_out/trip_scale.txt
  grep '^{' gpurun_out/trip_n$n.log >> gpurun_out/trip_scale.txt
done
cat gpurun_out/trip_scale.txt | cut -c1-400
