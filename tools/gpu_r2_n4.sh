#!/bin/bash
# 4 GPUs: configs[3] CCSD with samples (bitwise vs 1 GPU) and configs[4] strong with one row per tile pair
mkdir -p gpurun_out
timeout 2000 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/bench_ccsd.py --steps 1 --warmup 2 --ws-gb 12 --samples-out gpurun_out/r2q_ccsd_samples_n4.json > gpurun_out/r2q_ccsd_n4.jsonl 2> gpurun_out/r2q_ccsd_n4.err
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 tools/bench_cfg5.py --samples-out gpurun_out/r2q_cfg5_samples_strong_n4.json > gpurun_out/r2q_cfg5_n4.jsonl 2> gpurun_out/r2q_cfg5_n4.err
timeout 900 python tests/full_samples_check.py ccsd gpurun_out/r2q_ccsd_samples_n4.json > gpurun_out/r2q_check.log 2>&1
timeout 1500 python tests/full_samples_check.py cfg5 gpurun_out/r2q_cfg5_samples_strong_n4.json >> gpurun_out/r2q_check.log 2>&1
cat gpurun_out/r2q_check.log; grep '^{' gpurun_out/r2q_ccsd_n4.jsonl | head -c 300; echo; tail -c 800 gpurun_out/r2q_cfg5_n4.jsonl
