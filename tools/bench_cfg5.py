"""BASELINE configs[4]: large ladder R(a,b,i,j) += V(a,b,c,d) T(c,d,i,j) with the implicit
Cholesky-factored V of Eq. cc12 (never stored), O=150 V=1200 tile 64, alpha/beta spin maps,
N_L = 2(O+V), owner-computes over the GPUs of one box (torchrun, NCCL).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/bench_cfg5.py            # strong
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/bench_cfg5.py --weak     # weak

Placement: X replicated; T distributed over (c,d)-symmetric block pairs (T(c,d,i,j) and T(d,c,i,j) on
one rank, round robin over the pairs) with compact storage: each rank forms its half of
Bm = T - T(c<->d) from its own blocks and the half is all-gathered inside every call (the input-tile
gather of §8(e)); R split by (a,b) rows with tt_partition_split_cost on the executed cost of the
implicit ladder, compact.  The workspace holds that half of Bm plus W rows (--ws-gb 0: sized
automatically; too small a workspace selects the two-pass consume).  Weak scaling keeps the
per-GPU FLOPs constant: V = 714 / 848 / 1010 / 1200 for 1 / 2 / 4 / 8 GPUs.

Timing: W warm-up calls, then K calls bracketed by a barrier + CUDA events, max over ranks.
--samples-out writes sampled R elements (owned rows gathered on rank 0) for the CPU oracle check
tests/test_cfg5_samples.py; no oracle code runs here."""
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

WEAK_V = {1: 714, 2: 848, 4: 1010, 8: 1200}
ALPHA = 0.5
SEED = 1


def sample_positions(O, V, voffs, per_row=2, seed=11):
    """(a, b, i, j) global positions: one (a,b) row per (a_t, b_t) tile pair -- every tile pair of R,
    hence every R block row, is sampled -- at a seeded position inside the tiles,
    with ``per_row`` (i,j) columns of conserved spin each."""
    rng = np.random.default_rng(seed)
    h, o = V // 2, O // 2
    out = []
    nt = len(voffs) - 1
    for ta in range(nt):
        for tb in range(nt):
            a = int(rng.integers(voffs[ta], voffs[ta + 1]))
            b = int(rng.integers(voffs[tb], voffs[tb + 1]))
            sa, sb = a < h, b < h
            k = 0
            while k < per_row:
                i, j = int(rng.integers(0, O)), int(rng.integers(0, O))
                if (sa + sb) == ((i < o) + (j < o)):
                    out.append((a, b, i, j))
                    k += 1
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--O", type=int, default=150)
    ap.add_argument("--V", type=int, default=1200)
    ap.add_argument("--tile", type=int, default=64)
    ap.add_argument("--nl", type=int, default=0, help="0: 2(O+V)")
    ap.add_argument("--ltile", type=int, default=450)
    ap.add_argument("--ws-gb", type=float, default=0.0,
                    help="0: half of Bm + one W row + 1 GB, capped by the free memory (else two-pass)")
    ap.add_argument("--weak", action="store_true")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=2)   # >= 2: tt_contract autotunes on the first two calls
    ap.add_argument("--samples-out", default="")
    ap.add_argument("--lib-ws-gb", type=float, default=2.0, help="libtt device workspace (tt_workspace_bind)")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    t_start = time.time()

    def log(msg):
        if rank == 0:
            free, tot = torch.cuda.mem_get_info()
            print(f"[{time.time() - t_start:8.1f} s] {msg} (free {free / 1e9:.1f} of {tot / 1e9:.1f} GB)",
                  file=sys.stderr, flush=True)

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    nid = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [tt.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    O = a.O
    V = WEAK_V[world] if a.weak else a.V
    NL = a.nl or 2 * (O + V)
    stream = torch.cuda.current_stream()
    # library workspace (metadata of the 400k-task plans and of every batch of the implicit ladder)
    ctx = tt.Context(device=local, stream=stream.cuda_stream, rank=rank, nranks=world, nccl_id=nid,
                     workspace_bytes=int(a.lib_ws_gb * (1 << 30)))
    so = tt.IndexSpace(O, [(0, O // 2), (O // 2, O)], [1, -1])
    sv = tt.IndexSpace(V, [(0, V // 2), (V // 2, V)], [1, -1])
    to, tv = tt.TiledIndexSpace(so, a.tile), tt.TiledIndexSpace(sv, a.tile)
    tl = tt.TiledIndexSpace(tt.IndexSpace(NL), a.ltile)
    R = tt.Tensor(ctx, [tv, tv, to, to], spin=([0, 1], [2, 3]))
    T = tt.Tensor(ctx, [tv, tv, to, to], spin=([0, 1], [2, 3]))
    X = tt.Tensor(ctx, [tv, tv, tl], spin=([0], [1]))
    X.set_owner(np.where(X.nz > 0, tt.TT_REPLICATED, -1).astype(np.int32))
    if world > 1:
        tt.partition_split_cholesky(ctx, R, "abij", X, "abcd", T, "cdij", group_dims=(0, 1))
        R.set_compact(True)
        # T's (c,d) / (d,c) block pairs placed together, balanced by bytes (LPT over pair volumes)
        offs = [np.diff(d.offsets) for d in T.dims]
        pairs = {}
        for blk in np.flatnonzero(T.nz):
            c = list(np.unravel_index(blk, T.grid))
            key = (min(c[0], c[1]), max(c[0], c[1]), c[2], c[3])
            pairs.setdefault(key, []).append(int(blk))
        vol = {k: sum(int(np.prod([offs[d][x] for d, x in enumerate(np.unravel_index(b, T.grid))])) for b in v)
               for k, v in pairs.items()}
        load = np.zeros(world)
        own = np.full(T.nblocks, -1, np.int32)
        for k in sorted(pairs, key=lambda k: (-vol[k], k)):
            r = int(np.argmin(load))
            load[r] += vol[k]
            own[pairs[k]] = r
        T.set_owner(own)
        T.set_compact(True)
    sz = np.diff(tv.offsets)
    half = 0
    for blk in np.flatnonzero(T.nz):
        c = np.unravel_index(blk, T.grid)
        if c[0] <= c[1]:
            half += int(sz[c[0]] * sz[c[1]] * np.diff(to.offsets)[c[2]] * np.diff(to.offsets)[c[3]])
    wrow = int(sz.max() ** 2 * (V // 2) ** 2)
    bufs = {}
    for name, Tn, tag in (("R", R, 3), ("T", T, 5), ("X", X, 7)):
        bufs[name] = torch.empty(Tn.storage_elems, dtype=torch.float64, device="cuda")
        Tn.bind(bufs[name])
        tt.fill_synthetic(ctx, Tn, SEED, tag)
    if a.ws_gb <= 0:      # half of Bm (tile pairs c_t <= d_t of T's map) + the largest W row + 1 GB
        free = torch.tensor([torch.cuda.mem_get_info()[0] / 1e9 - 4.0], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(free, op=dist.ReduceOp.MIN)
        a.ws_gb = min((half + wrow) * 8e-9 + 1.0, float(free[0]))
        if a.ws_gb < (half + wrow) * 8e-9:
            a.ws_gb = min(a.ws_gb, wrow * 8e-9 + 1.0)    # two-pass consume: W rows only
    ws = torch.empty(int(a.ws_gb * 1e9 / 8), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    log(f"inputs filled, workspace {a.ws_gb:.1f} GB")
    for _ in range(a.warmup):
        tt.contract_cholesky(ctx, R, "abij", 0.0, ALPHA, X, "abcd", T, "cdij", ws)
        torch.cuda.synchronize()
        log("warm-up call done")
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        tt.contract_cholesky(ctx, R, "abij", 0.0, ALPHA, X, "abcd", T, "cdij", ws)
    e1.record(stream)
    torch.cuda.synchronize()
    st = ctx.stats()
    ms = e0.elapsed_time(e1) / a.steps
    v = torch.tensor([ms, st["flops"], st["aux_flops"], st["gathered_bytes"],
                      torch.cuda.max_memory_allocated() / 1e9], dtype=torch.float64, device="cuda")
    vmax = v.clone()
    if world > 1:
        dist.all_reduce(v)
        dist.all_reduce(vmax, op=dist.ReduceOp.MAX)
    ms_max = float(vmax[0])
    flops, aux = float(v[1]), float(v[2])
    # sampled outputs of the rows this rank owns
    samples = []
    if a.samples_out:
        offs = [tv.offsets, tv.offsets, to.offsets, to.offsets]
        for pos in sample_positions(O, V, [int(x) for x in tv.offsets]):
            t = [int(np.searchsorted(offs[d], pos[d], side="right") - 1) for d in range(4)]
            blk = int(np.ravel_multi_index(t, R.grid))
            loc = [pos[d] - int(offs[d][t[d]]) for d in range(4)]
            ext = [int(offs[d][t[d] + 1] - offs[d][t[d]]) for d in range(4)]
            e = int(np.ravel_multi_index(loc, ext))
            mine = R.owner[blk] == rank or (R.owner[blk] == tt.TT_SPLIT and any(
                bb == blk and lo <= loc[0] < hi and ow == rank for (bb, lo, hi, ow) in R.parts))
            if world == 1:
                mine = True
            if mine:
                samples.append([*pos, float(bufs["R"][int(R.storage_off[blk]) + e])])
        if world > 1:
            allv = [None] * world
            dist.all_gather_object(allv, samples)
            samples = [x for part in allv for x in part]
    if rank == 0:
        rec = {"workload": f"configs[4] ladder R(abij) += V(abcd) T(cdij), implicit Cholesky V (Eq. cc12), "
                           f"O={O} V={V} tile={a.tile} N_L={NL} (L tile {a.ltile}), alpha/beta maps",
               "scaling": "weak" if a.weak else "strong", "n_gpus": world, "ms_per_ladder": ms_max,
               "algorithmic_flops": flops, "tflops": flops / (ms_max * 1e-3) / 1e12,
               "pct_fp64_peak": flops / (ms_max * 1e-3) / 1e12 / 37.1 / world * 100,
               "executed_flops": aux, "executed_tflops": aux / (ms_max * 1e-3) / 1e12,
               "gathered_gb_total": float(v[3]) / 1e9, "max_mem_gb_per_rank": float(vmax[4]),
               "tensor_gb": {"R_packed": R.packed_elems * 8e-9, "R_storage_rank0": R.storage_elems * 8e-9,
                             "T": T.packed_elems * 8e-9, "X": X.packed_elems * 8e-9},
               "workspace_gb": a.ws_gb, "steps": a.steps, "warmup": a.warmup}
        print(json.dumps(rec), flush=True)
        if a.samples_out:
            with open(a.samples_out, "w") as f:
                json.dump({"O": O, "V": V, "tile": a.tile, "NL": NL, "ltile": a.ltile, "seed": SEED, "alpha": ALPHA,
                           "tags": {"R": 3, "T": 5, "X": 7}, "n_gpus": world, "samples": samples}, f)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    try:
        main()
    except Exception:     # do not leave the other ranks waiting in NCCL
        import traceback
        traceback.print_exc()
        sys.stderr.flush()
        os._exit(1)
