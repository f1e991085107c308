#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
timeout 600 python tools/bench_triples.py --steps 3 --cpu-triples 0 > gpurun_out/r2w_trip_$r.jsonl 2>&1
timeout 600 python tools/bench_triples.py --spin --steps 3 --cpu-triples 0 > gpurun_out/r2w_trip_spin_$r.jsonl 2>&1
done
B="python tools/bench_triples.py --O 24 --V 120 --steps 1 --warmup 1 --cpu-triples 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:triples_fused_tma -c 1 -o gpurun_out/r2w_trip $B > gpurun_out/r2w_ncu.log 2>&1
for f in gpurun_out/r2w_trip*.jsonl; do echo $f; grep -o '"ms_per_step": [0-9.]*\|"kernels_rank0[^}]*}[^}]*}' $f; done; tail -3 gpurun_out/r2w_ncu.log
