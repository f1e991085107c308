#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_elem_modes.py -q -m gpu > gpurun_out/r2e2_test.log 2>&1; echo rc=$? >> gpurun_out/r2e2_test.log
timeout 300 python tools/bench_elem.py --steps 10 > gpurun_out/r2e2_elem.jsonl 2>&1
tail -3 gpurun_out/r2e2_test.log; cat gpurun_out/r2e2_elem.jsonl
