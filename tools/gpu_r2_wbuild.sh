#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/sanitize_mini.py > gpurun_out/r2w_mini.log 2>&1; echo rc=$? >> gpurun_out/r2w_mini.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_next3.py tests/test_ccsd_iteration.py tests/test_workspace.py -q -m gpu -x > gpurun_out/r2w_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2w_pytest.log
timeout 900 python tools/bench_cholesky.py --ws-gb 40 --steps 1 --warmup 2 > gpurun_out/r2w_chol.jsonl 2>&1
tail -3 gpurun_out/r2w_mini.log gpurun_out/r2w_pytest.log; cat gpurun_out/r2w_chol.jsonl | tail -c 1200
