#!/bin/bash
# 4-GPU box: (T) strong scaling, configs[3] CCSD at 1 and 4 GPUs (samples rechecked), bench.py at N=2,4
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 600 $R --nproc-per-node $N --master-port 2961$N tools/bench_triples.py --steps 3 --cpu-triples 0 > gpurun_out/r2f_trip_n$N.jsonl 2>&1
done
timeout 600 $R --nproc-per-node 4 --master-port 29620 tools/bench_triples.py --spin --steps 3 --cpu-triples 0 > gpurun_out/r2f_trip_spin_n4.jsonl 2>&1
timeout 1500 python tools/bench_ccsd.py --steps 1 --warmup 2 --ws-gb 12 --samples-out gpurun_out/r2f_ccsd_samples_n1.json > gpurun_out/r2f_ccsd_n1.jsonl 2> gpurun_out/r2f_ccsd_n1.err
timeout 1500 $R --nproc-per-node 4 --master-port 29630 tools/bench_ccsd.py --steps 1 --warmup 2 --ws-gb 12 --samples-out gpurun_out/r2f_ccsd_samples_n4.json > gpurun_out/r2f_ccsd_n4.jsonl 2> gpurun_out/r2f_ccsd_n4.err
for N in 1 4; do timeout 900 python tests/full_samples_check.py ccsd gpurun_out/r2f_ccsd_samples_n$N.json >> gpurun_out/r2f_check.log 2>&1; done
for N in 2 4; do
  timeout 900 $R --nproc-per-node $N --master-port 2964$N bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/r2f_bench_n$N.jsonl 2> gpurun_out/r2f_bench_n$N.err
done
for f in gpurun_out/r2f_trip*.jsonl; do echo $f; grep -o '"ms_per_step": [0-9.]*\|"energy": [-0-9.e]*' $f | head -2; done
for f in gpurun_out/r2f_ccsd_n*.jsonl gpurun_out/r2f_bench_n*.jsonl; do echo $f; grep '^{' $f | head -c 300; echo; done
cat gpurun_out/r2f_check.log
