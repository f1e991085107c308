#!/bin/bash
# launch list and full capture with the variant the plain run's autotune picks (3), so that the
# per-kernel shares compare with the plain run; the autotune trials under ncu are distorted
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2m_launches.csv python bench.py --steps 3 --warmup 3 --variant 3 > gpurun_out/r2m_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tt_contract -s 3 -c 1 -o gpurun_out/r2m_contract python bench.py --steps 1 --warmup 3 --no-sub --variant 3 > gpurun_out/r2m_ncu2.log 2>&1
tail -n 1 gpurun_out/r2m_ncu2.log; grep -c gpu__time gpurun_out/r2m_launches.csv
