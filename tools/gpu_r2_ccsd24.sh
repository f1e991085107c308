#!/bin/bash
mkdir -p gpurun_out
for N in 2 4; do
  timeout 2000 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N tools/bench_ccsd.py --steps 1 --warmup 2 --ws-gb 12 --samples-out gpurun_out/r2cc_samples_n$N.json --terms-out gpurun_out/r2cc_terms_n$N.json > gpurun_out/r2cc_bench_n$N.jsonl 2> gpurun_out/r2cc_bench_n$N.err
  timeout 900 python tests/full_samples_check.py ccsd gpurun_out/r2cc_samples_n$N.json >> gpurun_out/r2cc_check.log 2>&1
done
cat gpurun_out/r2cc_check.log; for N in 2 4; do grep '^{' gpurun_out/r2cc_bench_n$N.jsonl | head -c 250; echo; done
