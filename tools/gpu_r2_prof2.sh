#!/bin/bash
mkdir -p gpurun_out
B="python tools/bench_triples.py --O 24 --V 120 --steps 1 --warmup 1 --cpu-triples 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:triples_fused_tma -c 1 -o gpurun_out/r2y_trip $B > gpurun_out/r2y_ncu.log 2>&1
timeout 900 python tools/bench_cholesky.py --ws-gb 40 --steps 1 --warmup 2 > gpurun_out/r2y_chol.jsonl 2>&1
C="python tools/bench_cholesky.py --V 400 --ws-gb 8 --steps 1 --warmup 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tt_contract_tma_kernel -c 1 -o gpurun_out/r2y_wbuild $C > gpurun_out/r2y_ncu2.log 2>&1
tail -2 gpurun_out/r2y_ncu.log gpurun_out/r2y_ncu2.log; tail -c 800 gpurun_out/r2y_chol.jsonl
