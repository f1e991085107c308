#!/bin/bash
# round 2: workspace ABI + full GPU suite
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_workspace.py -x -q -m gpu > gpurun_out/r2w_ws.log 2>&1; echo rc=$? >> gpurun_out/r2w_ws.log
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/r2w_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2w_pytest.log
(timeout 300 python __graft_entry__.py --smoke > gpurun_out/r2w_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/r2w_smoke.log)
tail -n 3 gpurun_out/r2w_*.log
