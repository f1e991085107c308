#!/bin/bash
mkdir -p gpurun_out
B="python tools/bench_triples.py --spin --steps 1 --warmup 1 --cpu-triples 0"
timeout 900 ncu --set full --clock-control none -k regex:triples_fused_tma -c 1 -o gpurun_out/r2h_trip_spin $B > gpurun_out/r2h_ncu.log 2>&1
B2="python tools/bench_triples.py --steps 1 --warmup 1 --cpu-triples 0"
timeout 900 ncu --set full --clock-control none -k regex:triples_fused_tma -c 1 -o gpurun_out/r2h_trip_dense $B2 > gpurun_out/r2h_ncu2.log 2>&1
tail -n 2 gpurun_out/r2h_ncu.log; tail -n 2 gpurun_out/r2h_ncu2.log
