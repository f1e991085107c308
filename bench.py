#!/usr/bin/env python
"""Benchmark of the hot path on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config cfg2|cfg3]

Default workload (the bench line the driver records): BASELINE.json configs[1], the CCSD
particle-particle ladder R(a,b,i,j) += V(a,b,c,d) * T(c,d,i,j), O=40 V=200 tile=40, FP64.
--config cfg3: configs[2], spin-block-sparse doubles terms ladder + ring + hole-hole, O=60 V=400,
tO=30 tV=40 with the alpha/beta block maps of DESIGN.md R7 (one step = all three contractions).

One step = the tt_contract call(s) of the workload over the whole tensors (task lists, partition and
gather plans cached; the input-tile gather over NCCL when N > 1; the DMMA contraction kernel).
value = algorithmic FLOPs of all ranks (non-zero tile pairs only) / max over ranks of the device
time of the K timed steps (CUDA events on the context stream).  The operands (V = 12.8 GB for cfg2,
76.8 GB for cfg3) are larger than L2 (126 MB), so no explicit L2 flush is needed between steps.

N > 1 (torchrun): strong scaling of the same problem.  Owner-computes: the R (a,b) rows are laid
along a cost axis and cut into equal shares (tt_partition_split: a row straddling a rank boundary is
split along a), the V blocks live with the R rows (or row parts) that read them, every other input is
distributed round robin (P210 scheme 3) and gathered with grouped NCCL send/recv every step -- all
terms' gathers are issued first on the communication stream (tt_contract_prefetch) so they overlap
the other terms' kernels.  The kernel tile variant is autotuned by tt_contract on its first two calls
(warm-up), with identical bits.

e2e: the same step from pinned host memory through the library's own end-to-end call tt_contract_host
(include/tt.h): N = 1 pipelines inside libtt (per (a, b) tile pair of R: H2D of the operand rows on the
library's copy stream overlaps the previous chunk's contraction, finished R rows go back while the next
computes; checked bit for bit against upload + step + download); N > 1: the same per rank over the
blocks / row parts it holds (T's remote blocks gathered over NVLink first), also checked bit for bit.

sub_configs (N = 1, default run): configs[0] (launch-latency bound: us per contraction, HBM fraction
of its compulsory bytes) and configs[2] (one step of its three terms, own roofline), measured after the
configs[1] line's timed region.

--impl reference: the CPU oracle (oracle/) on the host cores, on a bounded sample of the same
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
# FP64 tensor-core peak: register-only mma.sync m8n8k4 (DMMA.8x8x4) probe on this pool's B200,
# 148 SMs at 1964 MHz (profiles/r01_probe_fp64.jsonl).  MEASURED_PEAKS.json has no FP64 entry.
FP64_PEAK_TFLOPS = 37.1
FP64_PEAK_SOURCE = "measured DMMA probe profiles/r01_probe_fp64.jsonl (37.1 TF/s @1964 MHz; cuBLAS DGEMM 35.5)"

CONFIGS = {
    "cfg1": dict(O=4, V=8, tO=4, tV=4, spin=False, terms=("ring",),
                 workload="cfg1 single contraction C(a,b,i,j) += A(a,c,i,k)*B(c,b,k,j), O=4 V=8 tile=4, dense, FP64"),
    "cfg2": dict(O=40, V=200, tO=40, tV=40, spin=False, terms=("ladder",),
                 workload="cfg2 CCSD ladder R(a,b,i,j) += V(a,b,c,d)*T(c,d,i,j), O=40 V=200 tile=40, dense, FP64"),
    "cfg3": dict(O=60, V=400, tO=30, tV=40, spin=True, terms=("ladder", "ring", "hh"),
                 workload="cfg3 spin-sparse CCSD doubles: ladder R+=V(abcd)T(cdij), ring R+=T(acik)W(cbkj), "
                          "hole-hole R+=T(abkl)W(klij); O=60 V=400 tO=30 tV=40, alpha/beta maps (R7), FP64"),
}


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def load_traffic(cfg: str, variant: int):
    """dram bytes per launch of the contraction kernel from the committed ncu --set full capture."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return d.get(f"{cfg}/v{variant}")
    except Exception:
        return None


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


# --------------------------------------------------------------------------------------------- problem

def build_problem(tt, ctx, c):
    """Tensors and contraction terms of a CCSD-shaped config (maps per DESIGN.md R6/R7)."""
    O_, V_ = c["O"], c["V"]
    if c["spin"]:
        so = tt.IndexSpace(O_, [(0, O_ // 2), (O_ // 2, O_)], [1, -1])
        sv = tt.IndexSpace(V_, [(0, V_ // 2), (V_ // 2, V_)], [1, -1])
    else:
        so, sv = tt.IndexSpace(O_), tt.IndexSpace(V_)
    to, tv = tt.TiledIndexSpace(so, c["tO"]), tt.TiledIndexSpace(sv, c["tV"])
    sp = (lambda up, lo: (up, lo)) if c["spin"] else (lambda up, lo: None)
    T = {"R": tt.Tensor(ctx, [tv, tv, to, to], spin=sp([0, 1], [2, 3]))}
    ops = []
    if "ladder" in c["terms"]:
        T["V"] = tt.Tensor(ctx, [tv, tv, tv, tv], spin=sp([0, 1], [2, 3]))
        T["T"] = tt.Tensor(ctx, [tv, tv, to, to], spin=sp([0, 1], [2, 3]))
        ops.append(("R", "abij", "V", "abcd", "T", "cdij"))
    if "ring" in c["terms"]:
        T["Ta"] = tt.Tensor(ctx, [tv, tv, to, to], spin=sp([0, 1], [2, 3]))
        T["Wr"] = tt.Tensor(ctx, [tv, tv, to, to], spin=sp([2, 1], [0, 3]))
        ops.append(("R", "abij", "Ta", "acik", "Wr", "cbkj"))
    if "hh" in c["terms"]:
        T["Tb"] = tt.Tensor(ctx, [tv, tv, to, to], spin=sp([0, 1], [2, 3]))
        T["Wh"] = tt.Tensor(ctx, [to, to, to, to], spin=sp([0, 1], [2, 3]))
        ops.append(("R", "abij", "Tb", "abkl", "Wh", "klij"))
    return (so, sv, to, tv), T, ops


def distribute(tt, ctx, T, ops, np):
    """Owner-computes placement for N > 1: R by (a,b) rows with the balanced row-splitting partition
    (tt_partition_split, group dims a,b: a row straddling a rank boundary is cut along a), V with the
    R rows (or row parts) that read it; other inputs keep the default round-robin owners (P210)."""
    R = T["R"]
    c, cl, a, al, b, bl = ops[0]
    tt.partition_split(ctx, R, cl, T[a], al, T[b], bl, group_dims=(0, 1))
    if "V" in T:
        V = T["V"]
        whole, split = {}, {}
        for blk in range(R.nblocks):
            if R.nz[blk]:
                ta, tb = (int(x) for x in np.unravel_index(blk, R.grid)[:2])
                if R.owner[blk] >= 0:
                    whole[(ta, tb)] = int(R.owner[blk])
        for (blk, lo, hi, ow) in R.parts:
            ta, tb = (int(x) for x in np.unravel_index(blk, R.grid)[:2])
            split.setdefault((ta, tb), set()).add((lo, hi, ow))
        vo = np.full(V.nblocks, -1, np.int32)
        vparts = []
        for blk in range(V.nblocks):
            if not V.nz[blk]:
                continue
            ta, tb = (int(x) for x in np.unravel_index(blk, V.grid)[:2])
            if (ta, tb) in split:
                vparts += [(blk, lo, hi, ow) for (lo, hi, ow) in sorted(split[(ta, tb)])]
                vo[blk] = 0
            else:
                vo[blk] = whole.get((ta, tb), 0)
        V.set_owner(vo)
        if vparts:
            V.set_parts(vparts)


_T_CACHE = {}


def cpu_oracle_sample(c, a0: int = 0):
    """The oracle (as it stands) on a bounded sample of the workload: the ladder output rows
    R[a0, :, :, :] (all b, i, j; K = V^2 contracted pairs), dense loops over the masked operands.
    Returns (flops the oracle executes, seconds, threads)."""
    import numpy as np
    import synthetic as S
    from oracle import ops as O
    O_, V_ = c["O"], c["V"]
    key = (O_, V_)
    if key not in _T_CACHE:
        _T_CACHE[key] = S.dense((V_, V_, O_, O_), 11, 5)
    Tt = _T_CACHE[key]
    g = a0 * V_ ** 3 + np.arange(V_ ** 3)
    Vs = S.values(11, 4, g).reshape(1, V_, V_, V_)
    C0 = S.values(11, 3, a0 * V_ * O_ * O_ + np.arange(V_ * O_ * O_)).reshape(1, V_, O_, O_)
    t0 = time.perf_counter()
    O.contract(C0, "abij", Vs, "abcd", Tt, "cdij", 1.0, 1.0)
    dt = time.perf_counter() - t0
    flops = 2.0 * V_ * O_ * O_ * V_ * V_
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return flops, dt, threads


def sub_records(tt, ctx, stream, np, torch, peaks):
    """configs[0] and configs[2] measured in the same run (N = 1), each with its own roofline: the
    default line's value stays configs[1]'s.  configs[0] is launch-latency bound (reported in us per
    contraction and as a fraction of the HBM roofline on its compulsory bytes), configs[2] is one step
    of its three terms against the FP64 tensor-core peak."""
    out = {}
    for name, steps in (("cfg1", 200), ("cfg3", 3)):
        c = CONFIGS[name]
        keep, T, ops = build_problem(tt, ctx, c)
        bufs = {}
        tags = {"R": 3, "V": 4, "T": 5, "Ta": 1, "Wr": 2, "Tb": 6, "Wh": 7}
        for n, Tn in T.items():
            bufs[n] = torch.empty(Tn.packed_elems, dtype=torch.float64, device="cuda")
            Tn.bind(bufs[n])
            tt.fill_synthetic(ctx, Tn, 11, tags[n])
        stats = []
        for w in range(3):
            stats = []
            for (cc, cl, a, al, b, bl) in ops:
                tt.contract(ctx, T[cc], cl, 1.0, 1.0, T[a], al, T[b], bl)
                stats.append(ctx.stats())
        torch.cuda.synchronize()
        ctx.set_profiling(True)
        ctx.profile_reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            for (cc, cl, a, al, b, bl) in ops:
                tt.contract(ctx, T[cc], cl, 1.0, 1.0, T[a], al, T[b], bl)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        kms, kn = ctx.profile("tt_contract_dmma")
        ctx.set_profiling(False)
        flops = sum(st["flops"] for st in stats)
        byts = sum(st["bytes"] for st in stats)
        avg_k = kms / max(kn, 1)
        rec = {"workload": c["workload"], "ms_per_step": ms, "value": flops / (ms * 1e-3) / 1e9, "unit": "GFLOP/s",
               "flops_per_step": flops, "compulsory_bytes_per_step": byts, "steps": steps}
        if name == "cfg1":
            hbm = peaks.get("hbm_gbs") or 6533.5
            rec["us_per_contraction"] = ms * 1e3
            rec["kernel_us"] = avg_k * 1e3
            rec["roofline"] = {"bound": "hbm", "achieved": byts / (avg_k * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                               "frac": byts / (avg_k * 1e-3) / 1e9 / hbm, "traffic": None,
                               "note": "launch-latency bound: 32 KB per launch"}
        else:
            per_launch = flops / max(kn // steps, 1)
            ach = per_launch / (avg_k * 1e-3) / 1e12
            rec["roofline"] = {"bound": "tensor", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                               "frac": ach / FP64_PEAK_TFLOPS, "traffic": None, "kernel": "tt_contract_dmma",
                               "kernel_share_of_step": kms / steps / ms}
            rec["pct_fp64_peak"] = flops / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS * 100
        out[name] = rec
        del bufs, T
        torch.cuda.empty_cache()
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if "RANK" in os.environ:   # torchrun pins OMP_NUM_THREADS=1; rank 0 runs alone, so give it the host cores
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    from oracle import _lib
    _lib.build()
    c = CONFIGS[args.config]
    for _ in range(args.warmup):
        cpu_oracle_sample(c, 0)
    tot_f, tot_t, threads = 0.0, 0.0, 1
    for s in range(args.steps):
        f, dt, threads = cpu_oracle_sample(c, (s * 7) % c["V"])
        tot_f += f
        tot_t += dt
    value = tot_f / tot_t / 1e9
    sample = (f"one ladder output slice R[a,:,:,:] per step ({c['V']} of {c['V'] ** 2} (a,b) rows, "
              f"K={c['V'] ** 2}), {args.steps} steps, dense oracle loops")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_t / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": c["workload"], "sample": sample},
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
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg3"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the configs[0] / configs[2] sub-records")
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

    cfg = CONFIGS[args.config]
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
    keep, T, ops = build_problem(tt, ctx, cfg)
    if world > 1:
        distribute(tt, ctx, T, ops, np)
    bufs = {}
    tags = {"R": 3, "V": 4, "T": 5, "Ta": 1, "Wr": 2, "Tb": 6, "Wh": 7}
    for name, Tn in T.items():
        bufs[name] = torch.empty(Tn.packed_elems, dtype=torch.float64, device="cuda")
        Tn.bind(bufs[name])
        tt.fill_synthetic(ctx, Tn, 11, tags[name])
    torch.cuda.synchronize()

    def step():
        if world > 1 and os.environ.get("TT_BENCH_PREFETCH", "1") != "0":
            # every term's input gather on the comm stream first: they overlap the other terms' kernels
            for (c, cl, a, al, b, bl) in ops:
                tt.contract_prefetch(ctx, T[c], cl, 1.0, T[a], al, T[b], bl)
        for (c, cl, a, al, b, bl) in ops:
            tt.contract(ctx, T[c], cl, 1.0, 1.0, T[a], al, T[b], bl)

    stats = []
    for w in range(args.warmup):
        if w == args.warmup - 1:
            stats = []
            for (c, cl, a, al, b, bl) in ops:
                tt.contract(ctx, T[c], cl, 1.0, 1.0, T[a], al, T[b], bl)
                stats.append(ctx.stats())
        else:
            step()
    torch.cuda.synchronize()
    flops_rank = sum(s["flops"] for s in stats)
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
    terms = []
    for (c, cl, a, al, b, bl), st in zip(ops, stats):
        t_ms, t_n = ctx.profile(f"tt_contract_dmma[{cl}={al}*{bl}]")
        t_avg = t_ms / max(t_n, 1)
        terms.append({"term": f"{c}({cl}) += {a}({al}) * {b}({bl})", "flops": st["flops"], "tasks": st["tasks"],
                      "kernel_ms": t_avg, "tflops": st["flops"] / (t_avg * 1e-3) / 1e12 if t_avg > 0 else None,
                      "variant": st["kernel_variant"]})
    ctx.set_profiling(False)
    if world > 1:   # per-rank term times (load balance evidence) on stderr
        print(json.dumps({"rank": rank, "ms_per_step": ms / args.steps,
                          "term_ms": [round(t["kernel_ms"], 2) for t in terms],
                          "term_gflop": [round(t["flops"] / 1e9, 1) for t in terms]}), file=sys.stderr, flush=True)
    tot = torch.tensor([ms, flops_rank], dtype=torch.float64, device="cuda")
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

    # roofline of the dominant kernel (this rank): FLOPs per launch / average launch time
    launches_per_step = max(kern_n // args.steps, 1)
    avg_kernel_ms = kern_ms / max(kern_n, 1)
    achieved = (flops_rank / launches_per_step) / (avg_kernel_ms * 1e-3) / 1e12
    variant = stats[0]["kernel_variant"]
    roof = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP64_PEAK_TFLOPS,
            # dram bytes per launch from the committed ncu capture of this config and variant on ONE GPU;
            # null at N > 1 (a rank's launch is a part of the problem the capture did not measure)
            "traffic": load_traffic(args.config, variant) if world == 1 else None,
            "kernel": "tt_contract_dmma", "avg_kernel_ms": avg_kernel_ms,
            "kernel_share_of_step": kern_ms / args.steps / ms_per_step, "peak_source": FP64_PEAK_SOURCE,
            "algorithmic_bytes_per_step": sum(s["bytes"] for s in stats)}

    # end to end through the C ABI with host buffers (pinned), N GPUs: tt_contract_host per term -- the
    # library pipelines the host<->device copies with the contraction tiles (N = 1) or moves each rank's
    # held ranges (N > 1); the pipelined step is checked bit for bit against upload + step + download
    e2e = None
    if not args.no_e2e:
        hosts = {}
        for name, Tn in T.items():
            hosts[name] = torch.empty(Tn.packed_elems, dtype=torch.float64, pin_memory=True)
            Tn.download_ptr(hosts[name].data_ptr())
        torch.cuda.synchronize()
        last = len(ops) - 1

        def e2e_step():
            up = set()
            for k, (c, cl, a, al, b, bl) in enumerate(ops):
                hA = hosts[a] if a not in up else None
                hB = hosts[b] if b not in up else None
                tt.contract_host(ctx, T[c], cl, 1.0, 1.0, T[a], al, T[b], bl, hA, hB, hosts[c],
                                 c_in=(k == 0), c_out=(k == last))
                up |= {a, b}

        def e2e_step_plain():
            for name, Tn in T.items():
                Tn.upload_ptr(hosts[name].data_ptr())
            step()
            T["R"].download_ptr(hosts["R"].data_ptr())

        def held_bytes(Tn):
            own = 0
            parts = {}
            for (blk, lo, hi, ow) in Tn.parts:
                parts.setdefault(blk, []).append((lo, hi, ow))
            for blk in range(Tn.nblocks):
                if not Tn.nz[blk]:
                    continue
                ext = [int(d.offsets[t + 1] - d.offsets[t]) for d, t in zip(Tn.dims, np.unravel_index(blk, Tn.grid))]
                vol = int(np.prod(ext))
                if Tn.owner[blk] == rank or Tn.owner[blk] == tt.TT_REPLICATED:
                    own += vol
                elif blk in parts:
                    own += sum(hi - lo for (lo, hi, ow) in parts[blk] if ow == rank) * (vol // ext[0])
            return 8 * own

        h2d = sum(held_bytes(T[n]) for n in T)
        d2h = held_bytes(T["R"])
        if True:   # the library's pipelined step must reproduce upload + step + download bit for bit
            r0 = hosts["R"].clone()
            e2e_step_plain()
            torch.cuda.synchronize()
            ref = hosts["R"].clone()
            hosts["R"].copy_(r0)
            e2e_step()
            ctx.sync()
            if not torch.equal(hosts["R"], ref):
                raise RuntimeError("tt_contract_host step differs from upload + tt_contract + download")
            hosts["R"].copy_(r0)
        e2e_step()
        ctx.sync()
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
        io = torch.tensor([h2d, d2h], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(io)
        e2e = {"value": flops_all / (e_ms * 1e-3) / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(io[0]),
               "d2h_bytes_per_step": int(io[1]), "ms_per_step": e_ms, "steps": args.e2e_steps,
               "api": "tt_contract_host (include/tt.h)",
               "how": ("pipelined inside libtt: per (a, b) tile pair of R, H2D of the operand rows on the "
                       "library's copy stream overlapping the previous chunk's contraction, D2H of finished R rows "
                       "overlapping the next; PCIe floor 13.8 GB / 55.6 GB/s = 249 ms") if world == 1 else
                      ("each rank, pipelined inside libtt: H2D of T's held blocks and NVLink gather of the rest, "
                       "then per (a, b) tile pair the V rows it holds on the copy stream overlapping the previous "
                       "chunk's contraction, D2H of its finished R rows")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        f, dt, threads = cpu_oracle_sample(cfg, 0)
        reps = 1
        if dt < 5.0:   # aim for ~10-30 s of CPU work
            reps = max(1, min(8, int(15.0 / max(dt, 1e-3))))
            for r in range(1, reps):
                ff, dd, threads = cpu_oracle_sample(cfg, r)
                f += ff
                dt += dd
        sample = (f"{reps} ladder output slice(s) R[a,:,:,:], a=0..{reps - 1} (each {cfg['V']} (a,b) rows x "
                  f"{cfg['O'] ** 2} (i,j), K={cfg['V'] ** 2}), dense oracle loops")
        cpu = {"value": f / dt / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "oracle", "sample": sample,
               "seconds": dt}

    peaks = load_peaks()
    subs = None
    if world == 1 and not args.no_sub and args.config == "cfg2":
        del bufs, T
        torch.cuda.empty_cache()
        subs = sub_records(tt, ctx, stream, np, torch, peaks)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded splitmix64 counter generator over global indices, uniform [-1,1)",
            "config": {"workload": cfg["workload"], "flops_per_step": flops_all,
                       "tasks_per_step": sum(s["tasks"] for s in stats), "kernel_variant": variant,
                       "l2": "operands larger than L2 (126 MB); no flush",
                       "parallelism": f"owner-computes over {world} GPU(s), balanced row-split partition of R by (a,b) rows"},
            "pct_fp64_peak": value / world / (FP64_PEAK_TFLOPS * 1e3) * 100.0,
            "roofline": roof, "terms": terms, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "hbm_peak_gbs": peaks.get("hbm_gbs"),
            "sub_configs": subs,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
