"""Multi-GPU check of NEXT-3 (run under torchrun, NCCL): tt_contract3 (cc9) and a contraction over sliced
views, with the default round-robin owners (P210) on every tensor, so the intermediate and the operands
are gathered over NCCL.  Each rank's owned output blocks are summed over the ranks (every block has one
owner) and compared with the oracle (normwise 1e-11).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port 29534 tests/mgpu_next3_check.py
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2201_01257_b200 as tt  # noqa: E402
import synthetic as S  # noqa: E402
from oracle import layout as L  # noqa: E402
from oracle import ops as O  # noqa: E402
from tests.cases import oracle_objects, product_objects  # noqa: E402
from tests.test_next3 import cc9_problem  # noqa: E402


def owned_only(T, got, rank):
    out = np.zeros_like(got)
    for blk in range(T.nblocks):
        if T.nz[blk] and T.owner[blk] == rank:
            o = T.blk_off[blk]
            ext = [d.offsets[t + 1] - d.offsets[t] for d, t in zip(T.dims, np.unravel_index(blk, T.grid))]
            n = int(np.prod(ext))
            out[o:o + n] = got[o:o + n]
    return out


def allsum(x):
    t = torch.from_numpy(x).cuda()
    dist.all_reduce(t)
    return t.cpu().numpy()


def main():
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [tt.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = tt.Context(device=local, stream=torch.cuda.current_stream().cuda_stream, rank=rank, nranks=world,
                     nccl_id=obj[0])
    ok = True
    # --- contract3 (cc9), dense and spin
    for spin, shape in ((False, (8, 16, 4, 4)), (True, (12, 20, 3, 5))):
        pb = cc9_problem(*shape, spin)
        orc = oracle_objects(pb)
        P = product_objects(tt, ctx, pb)
        dense, keep = {}, []
        for name, tag in (("R", 3), ("v", 6), ("t", 5)):
            dense[name] = O.dense_masked(orc[name], S.dense(orc[name].shape, 2, tag))
            buf = torch.from_numpy(O.pack(orc[name], dense[name])).cuda()
            P[name].bind(buf)
            keep.append(buf)
        plan = tt.contract3(ctx, P["R"], "abij", 0.5, 0.25, P["v"], "efmn", P["t"], "efij", P["t"], "abmn")
        ws = torch.empty(plan["ws_elems"], dtype=torch.float64, device="cuda")
        tt.contract3(ctx, P["R"], "abij", 0.5, 0.25, P["v"], "efmn", P["t"], "efij", P["t"], "abmn", ws)
        got = allsum(owned_only(P["R"], P["R"].download(), rank))
        ctx.sync()
        ref = O.pack(orc["R"], O.contract3_naive(dense["R"], "abij", dense["v"], "efmn", dense["t"], "efij", dense["t"],
                                                 "abmn", 0.25, 0.5, cmask=O.nz_mask(orc["R"])))
        err = float(np.abs(got - ref).max() / np.abs(ref).max())
        ok &= err <= 1e-11
        if rank == 0:
            print(f"contract3 spin={spin} {shape}: err {err:.2e} gathered {ctx.stats()['gathered_bytes']}", flush=True)
    # --- views: C(i, a in "second") += A(i, x in "first") B(x, a in "second")
    K = tt.IndexSpace(40, [(0, 16), (16, 40)], names=["first", "second"])
    tK = tt.TiledIndexSpace(K, 8)
    M = tt.IndexSpace(30)
    tM = tt.TiledIndexSpace(M, sizes=[10, 20])
    A, B, C = tt.Tensor(ctx, [tM, tK]), tt.Tensor(ctx, [tK, tK]), tt.Tensor(ctx, [tM, tK])
    oK = L.tile_fixed(L.IndexSpace(40, [(0, 16, 0), (16, 40, 0)]), 8)
    oM = L.tile_custom(L.IndexSpace(30), [10, 20])
    oA, oB, oC = L.tensor_dense_map([oM, oK]), L.tensor_dense_map([oK, oK]), L.tensor_dense_map([oM, oK])
    DA, DB, DC = S.dense((30, 40), 3, 1), S.dense((40, 40), 3, 2), S.dense((30, 40), 3, 3)
    keep = []
    for T, oT, D in ((A, oA, DA), (B, oB, DB), (C, oC, DC)):
        b = torch.from_numpy(O.pack(oT, D)).cuda()
        T.bind(b)
        keep.append(b)
    Cv = C.view([tM, tK("second")])
    tt.contract(ctx, Cv, "ia", 1.0, 0.5, A.view([tM, tK("first")]), "ix", B.view([tK("first"), tK("second")]), "xa")
    got = allsum(owned_only(C, C.download(), rank))
    ctx.sync()
    ref = DC.copy()
    cs = O.slice_of(ref, [(0, 30), (16, 40)])
    cs[...] = O.contract(cs, "ia", O.slice_of(DA, [(0, 30), (0, 16)]), "ix", O.slice_of(DB, [(0, 16), (16, 40)]), "xa",
                         0.5, 1.0)
    err = float(np.abs(got - O.pack(oC, ref)).max() / np.abs(ref).max())
    ok &= err <= 1e-11
    if rank == 0:
        print(f"view contraction: err {err:.2e}", flush=True)
    # --- tt_contract_prefetch: the gather on the comm stream gives bitwise the same result
    res = []
    for pf in (False, True):
        cb = torch.from_numpy(O.pack(oC, DC)).cuda()
        C.bind(cb)
        keep.append(cb)
        if pf:
            tt.contract_prefetch(ctx, C, "ia", 1.0, A, "ix", B, "xa")
            tt.contract_prefetch(ctx, C, "ia", 0.0, A, "ix", B, "xa")   # a second plan (beta = 0) queued too
        tt.contract(ctx, C, "ia", 1.0, 0.5, A, "ix", B, "xa")
        tt.contract(ctx, C, "ia", 0.0, 1.5, A, "ix", B, "xa")
        res.append(C.download())
        ctx.sync()
    same = bool(np.array_equal(res[0], res[1]))
    ok &= same
    if rank == 0:
        print(f"prefetched gathers bitwise equal: {same}", flush=True)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("MGPU_NEXT3_CHECK PASS" if int(flag[0]) == 1 else "MGPU_NEXT3_CHECK FAIL", flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
