#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_elem_modes.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2e3_test.log 2>&1; echo rc=$? >> gpurun_out/r2e3_test.log
timeout 300 python tools/bench_elem.py --steps 10 > gpurun_out/r2e3_elem.jsonl 2>&1
tail -3 gpurun_out/r2e3_test.log; cut -c1-250 gpurun_out/r2e3_elem.jsonl
