#!/bin/bash
mkdir -p gpurun_out
B="python tools/bench_triples.py --O 24 --V 120 --steps 1 --warmup 1 --cpu-triples 0"
timeout 300 $B > gpurun_out/r2nt_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:triples_fused_tma -c 1 -o gpurun_out/r2nt_trip $B > gpurun_out/r2nt_ncu.log 2>&1
tail -2 gpurun_out/r2nt_plain.log; tail -3 gpurun_out/r2nt_ncu.log
