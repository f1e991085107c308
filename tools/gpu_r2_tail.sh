#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/r2t2_test.log 2>&1; echo rc=$? >> gpurun_out/r2t2_test.log
tail -n 4 gpurun_out/r2t2_test.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 2; do
  timeout 900 $R --nproc-per-node $N --master-port 2975$N bench.py --gpus $N --steps 10 --warmup 3 --no-sub --no-e2e > gpurun_out/r2t2_bench_n$N.jsonl 2> gpurun_out/r2t2_bench_n$N.err
  python -c "
import json
for l in open('gpurun_out/r2t2_bench_n$N.jsonl'):
    if l.startswith('{'): d=json.loads(l); print($N, d['value'], d['ms_per_step'], d['gpu_launches'], d['config'].get('kernel_variant'))
"
done
timeout 900 python bench.py --no-sub --no-e2e > gpurun_out/r2t2_bench_n1.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r2t2_bench_n1.jsonl'):
    if l.startswith('{'): d=json.loads(l); print(1, d['value'], d['ms_per_step'], d['gpu_launches'])
"
