#!/bin/bash
# Final check on a 4-GPU box: the whole GPU suite (multi-GPU scripts run with 4 ranks), smoke, and the
# bench at N = 1, 2, 4 (the driver's SCALE protocol).
mkdir -p gpurun_out
(timeout 300 python __graft_entry__.py --smoke > gpurun_out/f4_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/f4_smoke.log)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f4_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/f4_pytest.log
timeout 600 python bench.py > gpurun_out/f4_bench_n1.log 2>&1
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n bench.py --gpus $n > gpurun_out/f4_bench_n$n.log 2>&1
done
tail -2 gpurun_out/f4_smoke.log; tail -3 gpurun_out/f4_pytest.log
for n in 1 2 4; do grep '^{"metric' gpurun_out/f4_bench_n$n.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['value']), d['ms_per_step'], d.get('e2e',{}) and round(d['e2e']['value']))"; done
