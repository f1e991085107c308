#!/bin/bash
# bench cfg2 (default) + cfg3, then ncu full capture of the cfg2 contraction kernel (chosen variant).
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo rc=$? >> gpurun_out/bench_cfg2.log
timeout 900 python bench.py --config cfg3 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; echo rc=$? >> gpurun_out/bench_cfg3.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tt_contract -s 3 -c 1 -o gpurun_out/prof_contract_v5 $B > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$? >> gpurun_out/ncu_full.log
tail -c 600 gpurun_out/bench_cfg2.log; tail -c 1200 gpurun_out/bench_cfg3.log; tail -n 2 gpurun_out/ncu_full.log
