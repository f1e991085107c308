#!/bin/bash
# configs[4] at 4 GPUs: memory probe, weak point (V=1010, two-pass: Bm does not fit), strong point (V=1200).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,memory.used --format=csv > gpurun_out/mem_probe.txt 2>&1
python -c "import torch; f,t=torch.cuda.mem_get_info(); print('mem_get_info free', f, 'total', t)" >> gpurun_out/mem_probe.txt 2>&1
run() { local n=$1; shift; local tag=$1; shift
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n tools/bench_cfg5.py "$@" > gpurun_out/cfg5_$tag.log 2>&1
  echo rc=$? >> gpurun_out/cfg5_$tag.log; }
run 4 weak_n4 --weak --ws-gb 10 --samples-out gpurun_out/cfg5_samples_weak_n4.json
run 4 strong_n4 --ws-gb 14 --samples-out gpurun_out/cfg5_samples_strong_n4.json
