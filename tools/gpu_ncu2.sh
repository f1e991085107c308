#!/bin/bash
# ncu captures: default bench kernel (cfg2, chosen variant) and the Cholesky W-build kernel.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
C="python tools/bench_cholesky.py --O 40 --V 200 --tile 40 --nl 480 --ltile 240 --ws-gb 8"
timeout 300 $B > gpurun_out/plain_b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tt_contract -s 3 -c 1 -o gpurun_out/prof_cfg2_default $B > gpurun_out/ncu_b.log 2>&1
echo ncu_b=$? >> gpurun_out/ncu_b.log
timeout 300 $C > gpurun_out/plain_c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tt_contract -s 2 -c 1 -o gpurun_out/prof_wbuild $C > gpurun_out/ncu_c.log 2>&1
echo ncu_c=$? >> gpurun_out/ncu_c.log
tail -n 2 gpurun_out/ncu_b.log gpurun_out/ncu_c.log; tail -n 1 gpurun_out/plain_c.log
