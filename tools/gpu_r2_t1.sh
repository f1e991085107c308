#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_triples.py -q -m gpu > gpurun_out/r2t_test.log 2>&1; echo rc=$? >> gpurun_out/r2t_test.log
timeout 600 python tools/bench_triples.py > gpurun_out/r2t_trip.jsonl 2>&1
timeout 600 python tools/bench_triples.py --spin > gpurun_out/r2t_trip_spin.jsonl 2>&1
timeout 2000 python tools/bench_ccsd.py --steps 1 --warmup 2 --ws-gb 12 --samples-out gpurun_out/r2t_ccsd_samples_n1.json > gpurun_out/r2t_ccsd_n1.jsonl 2>&1
timeout 900 python tests/full_samples_check.py ccsd gpurun_out/r2t_ccsd_samples_n1.json > gpurun_out/r2t_check.log 2>&1
tail -3 gpurun_out/r2t_test.log; tail -c 700 gpurun_out/r2t_trip.jsonl; tail -c 700 gpurun_out/r2t_trip_spin.jsonl; cat gpurun_out/r2t_check.log
