#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_triples.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2x_test.log 2>&1; echo rc=$? >> gpurun_out/r2x_test.log
timeout 600 python tools/bench_triples.py --steps 3 --cpu-triples 0 > gpurun_out/r2x_trip.jsonl 2>&1
timeout 600 python tools/bench_triples.py --spin --steps 3 --cpu-triples 0 > gpurun_out/r2x_trip_spin.jsonl 2>&1
timeout 900 python bench.py > gpurun_out/r2x_bench.jsonl 2>gpurun_out/r2x_bench.err
tail -3 gpurun_out/r2x_test.log
for f in gpurun_out/r2x_trip*.jsonl; do echo $f; grep -o '"ms_per_step": [0-9.]*\|"energy": [-0-9.e]*\|"tt_triples_fused": {[^}]*}' $f; done
python - <<'P'
import json
for l in open('gpurun_out/r2x_bench.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d.get('value'), d.get('unit'), d.get('ms_per_step'), d.get('roofline'), d.get('config',{}).get('workload'))
P
