#!/usr/bin/env python
"""Benchmark of the hot path: BASELINE.json configs[1], the CCSD particle-particle ladder
R(a,b,i,j) += V(a,b,c,d) * T(c,d,i,j), O=40 V=200 tile=40, FP64, on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One step = one tt_contract call (task list and partition cached; input-tile gather over NCCL when
N > 1; the DMMA contraction kernel) over the whole tensor.  value = algorithmic FLOPs of all ranks
/ max over ranks of the device time (CUDA events on the context stream).  Inputs (V 12.8 GB) are
larger than L2 (126 MB), so no explicit L2 flush is needed between steps.

N > 1 (torchrun): strong scaling of the same problem.  Owner-computes: R blocks are LPT-partitioned
over the ranks, V blocks live with the R rows that read them, T blocks are distributed round robin
and each step gathers the T blocks a rank needs with grouped NCCL send/recv inside tt_contract.

--impl reference: the CPU oracle (oracle/) timed on the host cores on a bounded sample of the same
workload (rank 0 only), same metric and unit.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 GFLOP/s and % of FP64 TC peak, CCSD contractions at 1/2/4/8 B200"
O_, V_, TILE = 40, 200, 40
WORKLOAD = "cfg2 CCSD ladder R(a,b,i,j) += V(a,b,c,d)*T(c,d,i,j), O=40 V=200 tile=40, dense, FP64"
# FP64 tensor-core peak: register-only mma.sync m8n8k4 (DMMA.8x8x4) probe on this pool's B200,
# 148 SMs at 1964 MHz (profiles/r01_probe_fp64.jsonl).  MEASURED_PEAKS.json has no FP64 entry.
FP64_PEAK_TFLOPS = 37.1
FP64_PEAK_SOURCE = "measured DMMA probe profiles/r01_probe_fp64.jsonl (37.1 TF/s @1964 MHz; cuBLAS DGEMM 35.5)"


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.lines, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[2:6]):
                if v.lower() in ("active", "1"):
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples": len(sm)}


def build_problem(tt, ctx):
    so, sv = tt.IndexSpace(O_), tt.IndexSpace(V_)
    to, tv = tt.TiledIndexSpace(so, TILE), tt.TiledIndexSpace(sv, TILE)
    R = tt.Tensor(ctx, [tv, tv, to, to])
    V = tt.Tensor(ctx, [tv, tv, tv, tv])
    T = tt.Tensor(ctx, [tv, tv, to, to])
    return (so, sv, to, tv), R, V, T


_T_CACHE = None


def cpu_oracle_sample(rows_a: int = 1, a0: int = 0):
    """Oracle (as it stands) on a bounded sample: the R rows a in [a0, a0+rows_a) of the same ladder,
    all b, i, j, full K = 40000.  Returns (flops, seconds, threads)."""
    import numpy as np
    import synthetic as S
    from oracle import ops as O
    global _T_CACHE
    ga = np.arange(a0, a0 + rows_a)
    gV = S.values(11, 4, (ga[:, None] * V_ ** 3 + np.arange(V_ ** 3)[None, :]).reshape(-1)).reshape(rows_a, V_, V_, V_)
    if _T_CACHE is None:
        _T_CACHE = S.dense((V_, V_, O_, O_), 11, 5)
    T = _T_CACHE
    C0 = S.values(11, 3, (ga[:, None] * (V_ * O_ * O_) + np.arange(V_ * O_ * O_)[None, :]).reshape(-1))
    C0 = C0.reshape(rows_a, V_, O_, O_)
    t0 = time.perf_counter()
    O.contract(C0, "abij", gV, "abcd", T, "cdij", 1.0, 1.0)
    dt = time.perf_counter() - t0
    flops = 2.0 * rows_a * V_ * O_ * O_ * V_ * V_
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return flops, dt, threads


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np  # noqa: F401
    from oracle import _lib
    _lib.build()
    for _ in range(args.warmup):
        cpu_oracle_sample(1, 0)
    tot_f, tot_t = 0.0, 0.0
    threads = 1
    for s in range(args.steps):
        f, dt, threads = cpu_oracle_sample(1, (s * 7) % V_)
        tot_f += f
        tot_t += dt
    value = tot_f / tot_t / 1e9
    sample = f"R rows a=one value per step (200 of 40000 (a,b) rows, K=40000), {args.steps} steps"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_t / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "sample": sample},
            "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--variant", type=int, default=None, help="force a contraction kernel variant (TT_FORCE_VARIANT)")
    args = ap.parse_args()
    if args.variant is not None:
        os.environ["TT_FORCE_VARIANT"] = str(args.variant)
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2201_01257_b200 as tt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    nid = None
    if world > 1:
        obj = [tt.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    ctx = tt.Context(device=local, stream=stream.cuda_stream, rank=rank, nranks=world, nccl_id=nid)
    keep, R, V, T = build_problem(tt, ctx)
    if world > 1:
        own = tt.partition_lpt(ctx, R, "abij", V, "abcd", T, "cdij")
        R.set_owner(own)
        # V block (a,b,c,d) lives with the R block (a,b,0,0) that reads it (owner-computes)
        vo = np.empty(V.nblocks, np.int32)
        g = V_ // TILE
        for b in range(V.nblocks):
            ab = b // (g * g)
            vo[b] = own[ab]      # R grid is (g, g, 1, 1)
        V.set_owner(vo)
    bufs = {}
    for name, Tn, tag in (("R", R, 3), ("V", V, 4), ("T", T, 5)):
        bufs[name] = torch.empty(Tn.packed_elems, dtype=torch.float64, device="cuda")
        Tn.bind(bufs[name])
        tt.fill_synthetic(ctx, Tn, 11, tag)
    torch.cuda.synchronize()

    def step():
        tt.contract(ctx, R, "abij", 1.0, 1.0, V, "abcd", T, "cdij")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st = ctx.stats()
    flops_rank = st["flops"]
    if world > 1:
        dist.barrier()
    ctx.set_profiling(True)
    ctx.profile_reset()
    l0 = ctx.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = ctx.launches() - l0
    ms = e0.elapsed_time(e1)
    kern_ms, kern_n = ctx.profile("tt_contract_dmma")
    ctx.set_profiling(False)
    tot = torch.tensor([ms, flops_rank, kern_ms / max(kern_n, 1)], dtype=torch.float64, device="cuda")
    if world > 1:
        mx = tot.clone()
        dist.all_reduce(mx[:1], op=dist.ReduceOp.MAX)
        sm_ = tot.clone()
        dist.all_reduce(sm_[1:2], op=dist.ReduceOp.SUM)
        ms_max, flops_all = float(mx[0]), float(sm_[1])
    else:
        ms_max, flops_all = ms, flops_rank
    ms_per_step = ms_max / args.steps
    value = flops_all / (ms_per_step * 1e-3) / 1e9

    # roofline of the dominant kernel (this rank)
    avg_kernel_ms = kern_ms / max(kern_n, 1)
    achieved = flops_rank / (avg_kernel_ms * 1e-3) / 1e12
    roof = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None, "kernel": "tt_contract_dmma",
            "avg_kernel_ms": avg_kernel_ms, "kernel_share_of_step": avg_kernel_ms / ms_per_step,
            "peak_source": FP64_PEAK_SOURCE}

    # end to end through the C ABI with host buffers (pinned), N GPUs
    e2e = None
    if not args.no_e2e:
        hosts = {}
        for name, Tn in (("R", R), ("V", V), ("T", T)):
            hosts[name] = torch.empty(Tn.packed_elems, dtype=torch.float64, pin_memory=True)
            Tn.download_ptr(hosts[name].data_ptr())
        torch.cuda.synchronize()
        h2d = 8 * (R.packed_elems + V.packed_elems + T.packed_elems)
        d2h = 8 * R.packed_elems

        def e2e_step():
            for name, Tn in (("V", V), ("T", T), ("R", R)):
                Tn.upload_ptr(hosts[name].data_ptr())
            step()
            R.download_ptr(hosts["R"].data_ptr())

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        f1.record(stream)
        torch.cuda.synchronize()
        ems = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e_ms = float(ems[0]) / args.e2e_steps
        e2e = {"value": flops_all / (e_ms * 1e-3) / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d * world,
               "d2h_bytes_per_step": d2h * world, "ms_per_step": e_ms, "steps": args.e2e_steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        f, dt, threads = cpu_oracle_sample(1, 0)
        if dt < 5.0:   # aim for ~10-30 s of CPU work
            reps = max(1, min(8, int(15.0 / max(dt, 1e-3))))
            f, dt = 0.0, 0.0
            for r in range(reps):
                ff, dd, threads = cpu_oracle_sample(1, r)
                f += ff
                dt += dd
            sample = f"{reps} R slices a=0..{reps - 1} (each 200 (a,b) rows x 1600 (i,j), K=40000)"
        else:
            sample = "1 R slice a=0 (200 (a,b) rows x 1600 (i,j), K=40000)"
        cpu = {"value": f / dt / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "oracle", "sample": sample,
               "seconds": dt}

    if rank == 0:
        peaks = load_peaks()
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded splitmix64 counter generator over global indices, uniform [-1,1)",
            "config": {"workload": WORKLOAD, "flops_per_step": flops_all, "tasks": st["tasks"] * world,
                       "kernel_variant": st["kernel_variant"],
                       "l2": "inputs larger than L2 (V = 12.8 GB >> 126 MB); no flush",
                       "parallelism": f"owner-computes over {world} GPU(s), LPT partition of R blocks"},
            "pct_fp64_peak": value / world / (FP64_PEAK_TFLOPS * 1e3) * 100.0,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "hbm_peak_gbs": peaks.get("hbm_gbs"),
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
