#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_sim_ranks.py tests/test_ccsd_iteration.py -q -m gpu -k "cholesky or sim or ccsd" > gpurun_out/r2o_test.log 2>&1; echo rc=$? >> gpurun_out/r2o_test.log
timeout 900 python tools/bench_cholesky.py --ws-gb 40 --steps 1 --warmup 2 > gpurun_out/r2o_chol.jsonl 2>&1
timeout 900 python tools/bench_ccsd.py --steps 1 --warmup 2 --ws-gb 12 > gpurun_out/r2o_ccsd.jsonl 2>&1
tail -n 2 gpurun_out/r2o_test.log; tail -c 560 gpurun_out/r2o_chol.jsonl; echo
python -c "
import json
for l in open('gpurun_out/r2o_ccsd.jsonl'):
    if l.startswith('{'): d=json.loads(l); print('ccsd', d['ms_per_iteration'], d['kernel_ms_rank0'].get('tt_contract_dmma[abij=abcd*cdij]'))
"
