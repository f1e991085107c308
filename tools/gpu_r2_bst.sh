#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_sim_ranks.py tests/test_ccsd_iteration.py tests/test_workspace.py -q -m gpu -k "cholesky or Cholesky or sim or ccsd or workspace" > gpurun_out/r2b_test.log 2>&1; echo rc=$? >> gpurun_out/r2b_test.log
timeout 900 python tools/bench_cholesky.py --ws-gb 40 --steps 1 --warmup 2 > gpurun_out/r2b_chol.jsonl 2>&1
timeout 900 python tools/bench_cholesky.py --ws-gb 40 --steps 1 --warmup 2 --ltile 1800 > gpurun_out/r2b_chol_lt1800.jsonl 2>&1
tail -n 3 gpurun_out/r2b_test.log; tail -c 600 gpurun_out/r2b_chol.jsonl; echo; tail -c 600 gpurun_out/r2b_chol_lt1800.jsonl
