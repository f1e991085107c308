#!/bin/bash
# 4-GPU box after the host split: multi-GPU pytest, configs[4] strong with samples, CCSD multi-GPU check
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_multigpu.py -q -m gpu > gpurun_out/r2k_mgpu_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2k_mgpu_pytest.log
timeout 900 $R --nproc-per-node 2 --master-port 29581 tests/mgpu_ccsd_check.py > gpurun_out/r2k_mgpu_ccsd_n2.log 2>&1; echo rc=$? >> gpurun_out/r2k_mgpu_ccsd_n2.log
timeout 2400 $R --nproc-per-node 4 --master-port 29582 tools/bench_cfg5.py --samples-out gpurun_out/r2k_cfg5_samples_n4.json > gpurun_out/r2k_cfg5_n4.jsonl 2> gpurun_out/r2k_cfg5_n4.err
timeout 1500 python tests/full_samples_check.py cfg5 gpurun_out/r2k_cfg5_samples_n4.json > gpurun_out/r2k_check.log 2>&1
tail -n 3 gpurun_out/r2k_mgpu_pytest.log; tail -n 3 gpurun_out/r2k_mgpu_ccsd_n2.log; cat gpurun_out/r2k_check.log; grep '^{' gpurun_out/r2k_cfg5_n4.jsonl | head -c 600
