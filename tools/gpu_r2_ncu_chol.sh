#!/bin/bash
mkdir -p gpurun_out
B="python tools/bench_cholesky.py --V 400 --ws-gb 8 --steps 1 --warmup 1"
timeout 600 $B > gpurun_out/r2n_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tt_contract_tma_kernel -c 1 -o gpurun_out/r2n_wbuild $B > gpurun_out/r2n_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tt_contract_ws_kernel -c 1 -o gpurun_out/r2n_exch $B > gpurun_out/r2n_ncu2.log 2>&1
tail -2 gpurun_out/r2n_plain.log; tail -3 gpurun_out/r2n_ncu1.log gpurun_out/r2n_ncu2.log
