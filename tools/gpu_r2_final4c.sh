#!/bin/bash
# final 4-GPU box: bench at N=2/4 (driver launch form), multi-GPU pytest, configs[3] CCSD at 4 GPUs with samples
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 900 $R --nproc-per-node $N --master-port 2965$N bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/r2y_bench_n$N.jsonl 2> gpurun_out/r2y_bench_n$N.err
done
timeout 1200 python -m pytest tests/test_multigpu.py -q -m gpu > gpurun_out/r2y_mgpu.log 2>&1; echo rc=$? >> gpurun_out/r2y_mgpu.log
timeout 1500 $R --nproc-per-node 4 --master-port 29660 tools/bench_ccsd.py --steps 1 --warmup 2 --ws-gb 12 --samples-out gpurun_out/r2y_ccsd_samples_n4.json > gpurun_out/r2y_ccsd_n4.jsonl 2> gpurun_out/r2y_ccsd_n4.err
timeout 900 python tests/full_samples_check.py ccsd gpurun_out/r2y_ccsd_samples_n4.json > gpurun_out/r2y_check.log 2>&1
tail -n 2 gpurun_out/r2y_mgpu.log; cat gpurun_out/r2y_check.log
for N in 2 4; do python -c "
import json
for l in open('gpurun_out/r2y_bench_n$N.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print($N, d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'])
"; done
grep '^{' gpurun_out/r2y_ccsd_n4.jsonl | head -c 400
