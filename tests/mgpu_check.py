"""Multi-GPU parity check (run under torchrun, one process per GPU, NCCL).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port 29511 tests/mgpu_check.py

For spin-sparse ladder / ring / hole-hole terms: output blocks LPT-partitioned over the ranks, inputs
distributed round robin (P210 scheme 3); tt_contract gathers the needed input blocks over NCCL. The
owned result blocks of all ranks are assembled on rank 0 and compared (a) bitwise with the same
contraction on one GPU (reading R12: results independent of the rank count) and (b) with the CPU
oracle (normwise 1e-11).  Also the scalar all-reduce and the permuted add."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2201_01257_b200 as tt  # noqa: E402
import synthetic as S  # noqa: E402
from oracle import ops as O  # noqa: E402
from tests.cases import TensorSpec, ccsd_problem, oracle_objects, product_objects  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [tt.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    stream = torch.cuda.current_stream().cuda_stream
    ctx = tt.Context(device=local, stream=stream, rank=rank, nranks=world, nccl_id=obj[0])
    pb = ccsd_problem(24, 80, 12, 20, True)
    pb.tensors["Rt"] = TensorSpec("ijab", ("spin", [0, 1], [2, 3]))
    P = product_objects(tt, ctx, pb)
    single = tt.Context(device=local, stream=stream) if rank == 0 else None
    P1 = product_objects(tt, single, pb) if rank == 0 else None
    c0, cl0, a0, al0, b0, bl0 = pb.ops[0]
    if os.environ.get("MGPU_SPLIT", "1") == "1":
        tt.partition_split(ctx, P[c0], cl0, P[a0], al0, P[b0], bl0, group_dims=(0, 1))
        # scatter some V rows across ranks too (parts of the inputs are gathered by row ranges)
        vparts = []
        for blk in range(P["Ta"].nblocks):
            if P["Ta"].nz[blk] and blk % 3 == 0:
                e0 = int(np.diff(P["Ta"].dims[0].offsets)[np.unravel_index(blk, P["Ta"].grid)[0]])
                vparts += [(blk, 0, e0 // 2, blk % world), (blk, e0 // 2, e0, (blk + 1) % world)]
        P["Ta"].set_parts(vparts)
    else:
        own = tt.partition_lpt(ctx, P[c0], cl0, P[a0], al0, P[b0], bl0)
        P["R"].set_owner(own)
    print(f"rank {rank}: R parts {len(P['R'].parts)}, split blocks {sum(1 for o in P['R'].owner if o == tt.TT_SPLIT)}",
          flush=True)
    bufs = {}
    for name, tag in (("R", 3), ("Vv", 4), ("T", 5), ("Ta", 1), ("Wr", 2), ("Tb", 6), ("Wh", 7), ("Rt", 8)):
        bufs[name] = torch.full((P[name].packed_elems,), float("nan"), dtype=torch.float64, device="cuda")
        P[name].bind(bufs[name])
        tt.fill_synthetic(ctx, P[name], 3, tag)
        if rank == 0:
            b1 = torch.empty(P1[name].packed_elems, dtype=torch.float64, device="cuda")
            P1[name].bind(b1)
            bufs[name + "_1"] = b1
            tt.fill_synthetic(single, P1[name], 3, tag)
    ok = True
    for k, (c, cl, a, al, b, bl) in enumerate(pb.ops):
        tt.contract(ctx, P[c], cl, 1.0, 0.5 + k, P[a], al, P[b], bl)
        st = ctx.stats()
        if rank == 0:
            tt.contract(single, P1[c], cl, 1.0, 0.5 + k, P1[a], al, P1[b], bl)
        print(f"rank {rank} term {k}: c_blocks {st['c_blocks']} tasks {st['tasks']} gathered {st['gathered_bytes']} B",
              flush=True)
    tt.add(ctx, P["R"], "abij", 1.0, -0.25, P["Rt"], "ijab")
    if rank == 0:
        tt.add(single, P1["R"], "abij", 1.0, -0.25, P1["Rt"], "ijab")
    s_multi = tt.contract_scalar(ctx, 0.25, P["Ta"], "acik", P["R"], "acik")
    # implicit Cholesky ladder (NEXT-1) across ranks: X replicated, R2 row-split, T gathered
    so, sv = P["_keep"][1]["O"], P["_keep"][1]["V"]
    sL = tt.IndexSpace(10)
    tL = tt.TiledIndexSpace(sL, 5)
    X = tt.Tensor(ctx, [sv, sv, tL], spin=([0], [1]))
    X.set_owner(np.where(X.nz > 0, tt.TT_REPLICATED, -1).astype(np.int32))
    R2 = tt.Tensor(ctx, [sv, sv, so, so], spin=([0, 1], [2, 3]))
    tt.partition_split(ctx, R2, "abij", P["Vv"], "abcd", P["T"], "cdij", group_dims=(0, 1))
    xb = torch.empty(X.packed_elems, dtype=torch.float64, device="cuda")
    r2b = torch.full((R2.packed_elems,), float("nan"), dtype=torch.float64, device="cuda")
    X.bind(xb)
    R2.bind(r2b)
    tt.fill_synthetic(ctx, X, 3, 9)
    tt.fill_synthetic(ctx, R2, 3, 10)
    ws = torch.empty(P["T"].packed_elems + 32 + 40 ** 4 * 16, dtype=torch.float64, device="cuda")
    tt.contract_cholesky(ctx, R2, "abij", 1.0, 0.5, X, "abcd", P["T"], "cdij", ws)
    g2 = R2.download()
    ctx.sync()
    mine2 = np.zeros_like(g2)
    for blk in range(R2.nblocks):
        if not R2.nz[blk]:
            continue
        o = R2.blk_off[blk]
        ext = [d.offsets[t + 1] - d.offsets[t] for d, t in zip(R2.dims, np.unravel_index(blk, R2.grid))]
        n = int(np.prod(ext))
        if R2.owner[blk] == rank:
            mine2[o:o + n] = g2[o:o + n]
        inner = n // int(ext[0])
        for (bb, lo, hi, ow) in R2.parts:
            if bb == blk and ow == rank:
                mine2[o + lo * inner:o + hi * inner] = g2[o + lo * inner:o + hi * inner]
    t2 = torch.from_numpy(mine2).cuda()
    dist.all_reduce(t2)
    assembled2 = t2.cpu().numpy()
    # again with T's (c,d) / (d,c) blocks co-located and T, R compact: each rank forms its own half of
    # Bm = T - T(c<->d) and the half is all-gathered (T itself is never gathered)
    T3 = tt.Tensor(ctx, [sv, sv, so, so], spin=([0, 1], [2, 3]))
    own3 = np.full(T3.nblocks, -1, np.int32)
    for blk in range(T3.nblocks):
        if T3.nz[blk]:
            cc = list(np.unravel_index(blk, T3.grid))
            cc[0], cc[1] = min(cc[0], cc[1]), max(cc[0], cc[1])
            own3[blk] = int(np.ravel_multi_index(cc, T3.grid)) % world
    T3.set_owner(own3)
    T3.set_compact(True)
    R3 = tt.Tensor(ctx, [sv, sv, so, so], spin=([0, 1], [2, 3]))
    tt.partition_split(ctx, R3, "abij", P["Vv"], "abcd", P["T"], "cdij", group_dims=(0, 1))
    R3.set_compact(True)
    t3b = torch.empty(T3.storage_elems, dtype=torch.float64, device="cuda")
    r3b = torch.full((R3.storage_elems,), float("nan"), dtype=torch.float64, device="cuda")
    T3.bind(t3b)
    R3.bind(r3b)
    tt.fill_synthetic(ctx, T3, 3, 5)
    ws3 = torch.empty(T3.packed_elems + 32 + 40 ** 4 * 16, dtype=torch.float64, device="cuda")
    tt.contract_cholesky(ctx, R3, "abij", 0.0, 0.5, X, "abcd", T3, "cdij", ws3)
    st3 = ctx.stats()
    g3 = R3.download()
    ctx.sync()
    mine3 = np.zeros(R3.packed_elems)
    for blk in range(R3.nblocks):
        if not R3.nz[blk]:
            continue
        o, so3 = R3.blk_off[blk], R3.storage_off[blk]
        ext = [d.offsets[t + 1] - d.offsets[t] for d, t in zip(R3.dims, np.unravel_index(blk, R3.grid))]
        n = int(np.prod(ext))
        if R3.owner[blk] == rank:
            mine3[o:o + n] = g3[so3:so3 + n]
        inner = n // int(ext[0])
        for (bb, lo, hi, ow) in R3.parts:
            if bb == blk and ow == rank:
                mine3[o + lo * inner:o + hi * inner] = g3[so3 + lo * inner:so3 + hi * inner]
    t3 = torch.from_numpy(mine3).cuda()
    dist.all_reduce(t3)
    assembled3 = t3.cpu().numpy()
    print(f"rank {rank}: co-located Cholesky ladder, T storage {T3.storage_elems} of {T3.packed_elems}, "
          f"gathered {st3['gathered_bytes']} B", flush=True)
    torch.cuda.synchronize()
    got = P["R"].download()
    ctx.sync()
    mine = np.zeros_like(got)
    live = np.zeros(got.shape, dtype=bool)
    for blk in range(P["R"].nblocks):
        if not P["R"].nz[blk]:
            continue
        o = P["R"].blk_off[blk]
        ext = [d.offsets[t + 1] - d.offsets[t] for d, t in zip(P["R"].dims, np.unravel_index(blk, P["R"].grid))]
        n = int(np.prod(ext))
        live[o:o + n] = True
        if P["R"].owner[blk] == rank:
            mine[o:o + n] = got[o:o + n]
        inner = n // int(ext[0])
        for (bb, lo, hi, ow) in P["R"].parts:
            if bb == blk and ow == rank:
                mine[o + lo * inner:o + hi * inner] = got[o + lo * inner:o + hi * inner]
    tot = torch.from_numpy(mine).cuda()
    dist.all_reduce(tot)   # each element owned by exactly one rank: the sum assembles the tensor
    assembled = tot.cpu().numpy()
    if rank == 0:
        s_single = tt.contract_scalar(single, 0.25, P1["Ta"], "acik", P1["R"], "acik")
        ref1 = P1["R"].download()
        single.sync()
        bit = np.array_equal(assembled[live], ref1[live])
        print(f"world {world}: R bitwise equal to 1-GPU result: {bit}", flush=True)
        ok &= bit
        # oracle
        orc = oracle_objects(pb)
        dense = {n: O.dense_masked(orc[n], S.dense(orc[n].shape, 3, t)) for n, t in
                 (("R", 3), ("Vv", 4), ("T", 5), ("Ta", 1), ("Wr", 2), ("Tb", 6), ("Wh", 7), ("Rt", 8))}
        Rd = dense["R"]
        m = O.nz_mask(orc["R"])
        for k, (c, cl, a, al, b, bl) in enumerate(pb.ops):
            Rd = O.contract(Rd, cl, dense[a], al, dense[b], bl, 0.5 + k, 1.0, cmask=m)
        Rd = O.add(Rd, "abij", dense["Rt"], "ijab", -0.25, 1.0, cmask=m)
        ref = O.pack(orc["R"], Rd)
        err = np.abs(assembled[live] - ref[live]).max() / np.abs(ref[live]).max()
        so = O.scalar(dense["Ta"], "acik", Rd, "acik", 0.25)
        print(f"world {world}: normwise error vs oracle {err:.3e}; scalar multi {s_multi:.15e} single {s_single:.15e} "
              f"oracle {so:.15e}", flush=True)
        ok &= err <= 1e-11 and abs(s_multi - so) <= 1e-12 * abs(so) and abs(s_single - so) <= 1e-12 * abs(so)
        # Cholesky term vs oracle (V formed explicitly from X, Eq. cc12)
        from oracle import layout as Lo
        oX = Lo.tensor_spin([orc["Vv"].dims[0], orc["Vv"].dims[0], Lo.tile_fixed(Lo.IndexSpace(10), 5)], [0], [1])
        Xd = O.dense_masked(oX, S.dense(oX.shape, 3, 9))
        R2d = O.dense_masked(orc["R"], S.dense(orc["R"].shape, 3, 10))
        ref2 = O.pack(orc["R"], O.contract(R2d, "abij", O.cholesky_v(Xd), "abcd", dense["T"], "cdij", 0.5, 1.0,
                                           cmask=m))
        err2 = np.abs(assembled2[live] - ref2[live]).max() / np.abs(ref2[live]).max()
        print(f"world {world}: Cholesky ladder normwise error vs oracle {err2:.3e}", flush=True)
        ok &= err2 <= 1e-11
        ref3 = O.pack(orc["R"], O.contract(np.zeros_like(R2d), "abij", O.cholesky_v(Xd), "abcd", dense["T"], "cdij",
                                           0.5, 0.0, cmask=m))
        err3 = np.abs(assembled3[live] - ref3[live]).max() / np.abs(ref3[live]).max()
        print(f"world {world}: co-located compact Cholesky ladder normwise error vs oracle {err3:.3e}", flush=True)
        ok &= err3 <= 1e-11
        print("MGPU_CHECK", "PASS" if ok else "FAIL", flush=True)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
