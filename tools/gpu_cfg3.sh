#!/bin/bash
mkdir -p gpurun_out
for v in "$@"; do
  timeout 900 python bench.py --config cfg3 --steps 3 --no-e2e --no-cpu-baseline --variant $v > gpurun_out/bench_cfg3_v$v.log 2>&1
  python -c "
import json,sys
l=[x for x in open('gpurun_out/bench_cfg3_v$v.log') if x.startswith('{')]
d=json.loads(l[-1]); print('v$v', round(d['value']), round(d['pct_fp64_peak'],2), [ (t['term'][:30], round(t['kernel_ms'],1), round(t['tflops'],2)) for t in d['terms']])" || tail -5 gpurun_out/bench_cfg3_v$v.log
done
