"""Perturbative triples (T) energy (PAPER Eq. cc14, P343-413) on 1..N GPUs.

    python tools/bench_triples.py [--O 40 --V 200 --tO 4 --tV 20 --ws-gb 40 --spin]
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/bench_triples.py

Inputs seeded synthetic (device fill by global index, identical on every rank; orbital energies
eps_o in (-2,-1), eps_v in (1,2)), replicated on every rank; the W tile triples are partitioned (LPT).
One step = the whole tt_triples_energy call (re-tiling, 18 contractions per batch, energy kernel,
all-reduce).  Reports the step time (max over ranks), the algorithmic FLOPs (the 18 terms over the
restricted a<b<c, i<j<k elements) and the executed FLOPs (whole tile triples), per-kernel times."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2201_01257_b200 as tt  # noqa: E402

INPUTS = [("T1", "vo", ([0], [1]), 11), ("T2", "vvoo", ([0, 1], [2, 3]), 12), ("Vooov", "ooov", ([0, 1], [2, 3]), 13),
          ("Vvovv", "vovv", ([0, 1], [2, 3]), 14), ("Voovv", "oovv", ([0, 1], [2, 3]), 15)]


def build(ctx, nO, nV, tO, tV, spin, world, seed=1):
    if spin:
        O = tt.IndexSpace(nO, [(0, nO // 2), (nO // 2, nO)], [1, -1])
        V = tt.IndexSpace(nV, [(0, nV // 2), (nV // 2, nV)], [1, -1])
    else:
        O, V = tt.IndexSpace(nO), tt.IndexSpace(nV)
    to, tv = tt.TiledIndexSpace(O, tO), tt.TiledIndexSpace(V, tV)
    dims = {"o": to, "v": tv}
    T, bufs = {}, []
    for n, d, sp, tag in INPUTS:
        T[n] = tt.Tensor(ctx, [dims[c] for c in d], spin=sp if spin else None)
        if world > 1:
            T[n].set_owner(np.full(T[n].nblocks, tt.TT_REPLICATED, np.int32))
        buf = torch.empty(max(T[n].storage_elems, 2), dtype=torch.float64, device="cuda")
        T[n].bind(buf)
        tt.fill_synthetic(ctx, T[n], seed, tag)
        bufs.append(buf)
    rng = np.random.default_rng(seed)
    eo = torch.from_numpy(rng.uniform(-2, -1, nO)).cuda()
    ev = torch.from_numpy(rng.uniform(1, 2, nV)).cuda()
    return T, (O, V, to, tv), bufs, eo, ev


def cpu_baseline(nO, nV, ntrip):
    """The oracle as it stands (oracle/triples.py energy_by_triple, numpy/BLAS on the host cores) on a
    bounded sample: the first ``ntrip`` occupied triples, every a<b<c; algorithmic FLOPs 18 (n_o + n_v)
    per restricted element (values are random: only the time matters)."""
    from oracle import triples as TR
    rng = np.random.default_rng(0)
    args = (rng.uniform(-1, 1, (nV, nO)), rng.uniform(-1, 1, (nV, nV, nO, nO)), rng.uniform(-1, 1, (nO, nO, nO, nV)),
            rng.uniform(-1, 1, (nV, nO, nV, nV)), rng.uniform(-1, 1, (nO, nO, nV, nV)), rng.uniform(-2, -1, nO),
            rng.uniform(1, 2, nV))
    t0 = time.time()
    _, n = TR.energy_by_triple(*args, max_triples=ntrip)
    dt = time.time() - t0
    flops = 18.0 * (nO + nV) * n
    return {"value": flops / dt / 1e9, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"{ntrip} occupied triples x all a<b<c ({n} elements), oracle by-triple form", "seconds": dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--O", type=int, default=40)
    ap.add_argument("--V", type=int, default=200)
    ap.add_argument("--tO", type=int, default=4)
    ap.add_argument("--tV", type=int, default=20)
    ap.add_argument("--spin", action="store_true")
    ap.add_argument("--ws-gb", type=float, default=40.0)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--cpu-triples", type=int, default=3,
                    help="occupied triples of the CPU oracle sample (rank 0, N=1; 0 = skip)")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    nid = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [tt.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    stream = torch.cuda.current_stream()
    ctx = tt.Context(device=local, stream=stream.cuda_stream, rank=rank, nranks=world, nccl_id=nid)
    t0 = time.time()
    T, keep, bufs, eo, ev = build(ctx, a.O, a.V, a.tO, a.tV, a.spin, world)
    args = (T["T1"], T["T2"], T["Vooov"], T["Vvovv"], T["Voovv"])
    _, q = tt.triples_energy(ctx, *args)
    ws = torch.empty(max(int(a.ws_gb * 1e9 / 8), q["ws_elems"]), dtype=torch.float64, device="cuda")
    E, info = tt.triples_energy(ctx, *args, eo, ev, ws)   # plans + first run
    setup_s = time.time() - t0
    for _ in range(a.warmup):
        tt.triples_energy(ctx, *args, eo, ev, ws)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ctx.set_profiling(True)
    ctx.profile_reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        E, info = tt.triples_energy(ctx, *args, eo, ev, ws)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    kernels = {}
    for name in ["tt_triples_fused", "tt_triples_blockify", "tt_retile", "tt_scalar_final"]:
        kms, kn = ctx.profile(name)
        kernels[name] = {"ms": round(kms / a.steps, 3), "launches": kn // a.steps}
    ctx.set_profiling(False)
    t = torch.tensor([ms, info["flops_exec"], info["flops_alg"]], dtype=torch.float64, device="cuda")
    if world > 1:
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        ms = float(mx[0])
    else:
        ms = float(t[0])
    cpu = None
    if rank == 0 and world == 1 and a.cpu_triples > 0:
        cpu = cpu_baseline(a.O, a.V, a.cpu_triples)
    if rank == 0:
        fexec, falg = float(t[1]), float(t[2])
        print(json.dumps({
            "workload": f"(T) energy O={a.O} V={a.V} tO={a.tO} tV={a.tV} {'alpha/beta maps' if a.spin else 'dense'}",
            "n_gpus": world, "ms_per_step": ms, "energy": E, "algorithmic_flops": falg, "executed_flops": fexec,
            "alg_tflops": falg / ms / 1e9, "exec_tflops": fexec / ms / 1e9,
            "pct_fp64_peak_executed": fexec / ms / 1e9 / 37.1 / world * 100,
            "w_blocks_total": info["w_blocks_total"], "w_blocks_rank0": info["w_blocks"],
            "batches_rank0": info["batches"], "kernels_rank0": kernels, "setup_s": round(setup_s, 1),
            "workspace_gb": ws.numel() * 8e-9, "cpu_baseline": cpu}), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
