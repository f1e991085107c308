#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k "contract_host" -q -m gpu > gpurun_out/r2b_test.log 2>&1; echo rc=$? >> gpurun_out/r2b_test.log
timeout 900 python bench.py > gpurun_out/r2b_bench.log 2>&1; echo rc=$? >> gpurun_out/r2b_bench.log
tail -3 gpurun_out/r2b_test.log; tail -c 4000 gpurun_out/r2b_bench.log
