#!/bin/bash
# round-2 launch list of the default bench command + one full capture of the headline kernel
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2l_plain.jsonl 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2l_launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/r2l_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tt_contract -s 3 -c 1 -o gpurun_out/r2l_contract python bench.py --steps 1 --warmup 3 --no-sub > gpurun_out/r2l_ncu2.log 2>&1
tail -n 2 gpurun_out/r2l_ncu.log; tail -n 2 gpurun_out/r2l_ncu2.log; grep -c gpu__time gpurun_out/r2l_launches.csv
