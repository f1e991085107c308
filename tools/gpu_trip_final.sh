#!/bin/bash
# (T): dense strong scaling on 1/2/4 GPUs, alpha/beta maps on 1 and 4 GPUs, ncu capture of the kernel
mkdir -p gpurun_out
rm -f gpurun_out/trip_final.txt
for n in 1 2 4; do
  if [ $n == 1 ]; then timeout 600 python tools/bench_triples.py > gpurun_out/tf_n$n.log 2>&1
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29541 tools/bench_triples.py > gpurun_out/tf_n$n.log 2>&1; fi
  grep '^{' gpurun_out/tf_n$n.log >> gpurun_out/trip_final.txt
done
timeout 600 python tools/bench_triples.py --spin > gpurun_out/tf_s1.log 2>&1; grep '^{' gpurun_out/tf_s1.log >> gpurun_out/trip_final.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 tools/bench_triples.py --spin > gpurun_out/tf_s4.log 2>&1; grep '^{' gpurun_out/tf_s4.log >> gpurun_out/trip_final.txt
B="python tools/bench_triples.py --O 24 --V 120 --steps 1 --warmup 0 --ws-gb 4 --cpu-triples 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:triples_fused -c 1 -o gpurun_out/prof_trip4 $B > gpurun_out/ncu_trip4.log 2>&1
echo ncu_rc=$? >> gpurun_out/trip_final.txt
cut -c1-300 gpurun_out/trip_final.txt
