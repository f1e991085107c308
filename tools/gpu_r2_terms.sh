#!/bin/bash
mkdir -p gpurun_out
N=${1:-4}
if [ "$N" == "1" ]; then
  timeout 2000 python tools/bench_ccsd.py --steps 1 --warmup 2 --ws-gb 12 --terms-out gpurun_out/r2t_terms_n1.json > gpurun_out/r2t_terms_n1.jsonl 2>&1
else
  timeout 2000 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29581 tools/bench_ccsd.py --steps 1 --warmup 2 --ws-gb 12 --terms-out gpurun_out/r2t_terms_n$N.json > gpurun_out/r2t_terms_n$N.jsonl 2>&1
fi
python -c "
import json; r=json.load(open('gpurun_out/r2t_terms_n$N.json')); print('serial', r['serial_ms_rank0'], 'scheduled', r['scheduled_ms'])
for t in sorted(r['terms'], key=lambda t: -t['ms_max_rank'])[:14]: print(t['ms_max_rank'], t['ms_rank0'], t['term'])
"
