#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_sim_ranks.py tests/test_ccsd_iteration.py -q -m gpu -k "cholesky or sim or ccsd" > gpurun_out/r2r_test.log 2>&1; echo rc=$? >> gpurun_out/r2r_test.log
TT_DEBUG=1 timeout 900 python tools/bench_ccsd.py --steps 1 --warmup 0 --ws-gb 12 > /dev/null 2> gpurun_out/r2r_dbg.err
timeout 900 python tools/bench_cholesky.py --ws-gb 40 --steps 1 --warmup 2 > gpurun_out/r2r_chol.jsonl 2>&1
tail -n 2 gpurun_out/r2r_test.log; grep -h "batches\|BsT" gpurun_out/r2r_dbg.err | head -2; tail -c 500 gpurun_out/r2r_chol.jsonl
