#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/bench_elem.py --steps 10 > gpurun_out/r2x_elem.jsonl 2>&1
timeout 600 python tools/bench_triples.py > gpurun_out/r2x_trip.jsonl 2>&1
timeout 600 python tools/bench_triples.py --spin > gpurun_out/r2x_trip_spin.jsonl 2>&1
cat gpurun_out/r2x_elem.jsonl; tail -c 1500 gpurun_out/r2x_trip.jsonl; tail -c 1500 gpurun_out/r2x_trip_spin.jsonl
