#!/bin/bash
# configs[4] strong scaling at N GPUs with one sampled row per (a_t, b_t) tile pair + host recheck
mkdir -p gpurun_out
N=${1:-4}
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29563 tools/bench_cfg5.py --samples-out gpurun_out/r2f_cfg5_samples_strong_n$N.json > gpurun_out/r2f_cfg5_n$N.jsonl 2> gpurun_out/r2f_cfg5_n$N.err
timeout 1800 python tests/full_samples_check.py cfg5 gpurun_out/r2f_cfg5_samples_strong_n$N.json > gpurun_out/r2f_check_n$N.log 2>&1
cat gpurun_out/r2f_check_n$N.log; grep '^{' gpurun_out/r2f_cfg5_n$N.jsonl | tail -c 900; grep -v "^\*\|OMP\|Warn" gpurun_out/r2f_cfg5_n$N.err | tail -3
