#!/bin/bash
mkdir -p gpurun_out
TT_DEBUG=1 timeout 900 python tools/bench_ccsd.py --steps 1 --warmup 0 --ws-gb 12 > gpurun_out/r2q_dbg_on.jsonl 2> gpurun_out/r2q_dbg_on.err
TT_CHOL_BST=0 TT_DEBUG=1 timeout 900 python tools/bench_ccsd.py --steps 1 --warmup 0 --ws-gb 12 > gpurun_out/r2q_dbg_off.jsonl 2> gpurun_out/r2q_dbg_off.err
timeout 900 python tools/bench_ccsd.py --steps 1 --warmup 2 --ws-gb 12 > gpurun_out/r2q_on.jsonl 2>&1
TT_CHOL_BST=0 timeout 900 python tools/bench_ccsd.py --steps 1 --warmup 2 --ws-gb 12 > gpurun_out/r2q_off.jsonl 2>&1
grep -h "batches\|BsT" gpurun_out/r2q_dbg_on.err | head -4; grep -h "batches\|BsT" gpurun_out/r2q_dbg_off.err | head -4
for f in on off; do python -c "
import json
for l in open('gpurun_out/r2q_$f.jsonl'):
    if l.startswith('{'): d=json.loads(l); print('$f', d['ms_per_iteration'], d['kernel_ms_rank0'].get('tt_contract_dmma[abij=abcd*cdij]'), d['kernel_ms_rank0'].get('tt_contract_dmma'))
"; done
