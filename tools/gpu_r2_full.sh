#!/bin/bash
# full GPU suite + smoke + default bench (the driver's round-end sequence)
mkdir -p gpurun_out
(timeout 300 python __graft_entry__.py --smoke > gpurun_out/r2z_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/r2z_smoke.log)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2z_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2z_pytest.log
timeout 900 python bench.py > gpurun_out/r2z_bench.log 2>&1; echo bench_rc=$? >> gpurun_out/r2z_bench.log
tail -n 3 gpurun_out/r2z_smoke.log gpurun_out/r2z_pytest.log; tail -c 1500 gpurun_out/r2z_bench.log
