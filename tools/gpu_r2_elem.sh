#!/bin/bash
# round 2: element-op per-descriptor modes + faster permuted kernels
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2e_smi.txt
timeout 900 python -m pytest tests/test_elem_modes.py tests/test_gpu_parity.py tests/test_ccsd_iteration.py -x -q -m gpu > gpurun_out/r2e_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2e_pytest.log
timeout 300 python tools/bench_elem.py --steps 10 > gpurun_out/r2e_elem.jsonl 2>&1
