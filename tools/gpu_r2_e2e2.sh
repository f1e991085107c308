#!/bin/bash
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $R --nproc-per-node 2 --master-port 29591 bench.py --gpus 2 --steps 10 --warmup 3 --no-sub > gpurun_out/r2e2_bench_n2.jsonl 2> gpurun_out/r2e2_bench_n2.err
timeout 900 python -m pytest tests/test_multigpu.py -q -m gpu > gpurun_out/r2e2_mgpu.log 2>&1; echo rc=$? >> gpurun_out/r2e2_mgpu.log
tail -n 2 gpurun_out/r2e2_mgpu.log; tail -n 3 gpurun_out/r2e2_bench_n2.err
python -c "
import json
for l in open('gpurun_out/r2e2_bench_n2.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])
"
