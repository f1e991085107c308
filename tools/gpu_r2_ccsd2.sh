#!/bin/bash
# textbook CCSD at configs[3] scale with full-size samples (and their CPU recheck on rank 0)
mkdir -p gpurun_out
N=${1:-1}; WS=${2:-4}
nproc > gpurun_out/r2cs_host.txt; free -g >> gpurun_out/r2cs_host.txt
if [ "$N" == "1" ]; then
  timeout 2400 python tools/bench_ccsd.py --steps 1 --warmup 2 --ws-gb $WS --samples-out gpurun_out/r2cs_samples_n1.json > gpurun_out/r2cs_bench_n1.jsonl 2> gpurun_out/r2cs_bench_n1.err
else
  timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29557 tools/bench_ccsd.py --steps 1 --warmup 2 --ws-gb $WS --samples-out gpurun_out/r2cs_samples_n$N.json > gpurun_out/r2cs_bench_n$N.jsonl 2> gpurun_out/r2cs_bench_n$N.err
fi
tail -c 600 gpurun_out/r2cs_bench_n$N.jsonl; tail -5 gpurun_out/r2cs_bench_n$N.err
