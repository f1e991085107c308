#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_triples.py -q -m gpu > gpurun_out/r2v_test.log 2>&1; echo rc=$? >> gpurun_out/r2v_test.log
timeout 300 python tools/bench_triples.py --O 12 --V 60 > gpurun_out/r2v_small.jsonl 2>&1
timeout 600 python tools/bench_triples.py > gpurun_out/r2v_trip.jsonl 2>&1
timeout 600 python tools/bench_triples.py --spin > gpurun_out/r2v_trip_spin.jsonl 2>&1
tail -3 gpurun_out/r2v_test.log; tail -c 600 gpurun_out/r2v_small.jsonl; tail -c 900 gpurun_out/r2v_trip.jsonl; tail -c 900 gpurun_out/r2v_trip_spin.jsonl
