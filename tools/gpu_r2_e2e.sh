#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "host" > gpurun_out/r2e_test.log 2>&1; echo rc=$? >> gpurun_out/r2e_test.log
timeout 900 python bench.py --no-sub > gpurun_out/r2e_bench.jsonl 2>&1
tail -n 2 gpurun_out/r2e_test.log
python -c "
import json
for l in open('gpurun_out/r2e_bench.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['e2e'])
"
