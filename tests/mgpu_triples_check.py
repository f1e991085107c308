"""Multi-GPU check of the (T) energy (run under torchrun, NCCL): inputs replicated on every rank (or
owner-distributed: round-robin owners, blocks held elsewhere NaN, gathered by each rank), units
split over the ranks, the partial energies all-reduced; compared with the oracle (by-triple form) and
with a 1-rank context on the same GPU (the same units summed in one place).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port 29533 tests/mgpu_triples_check.py
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
from oracle import triples as TR  # noqa: E402

INPUTS = [("T1", "vo", ([0], [1]), 11), ("T2", "vvoo", ([0, 1], [2, 3]), 12), ("Vooov", "ooov", ([0, 1], [2, 3]), 13),
          ("Vvovv", "vovv", ([0, 1], [2, 3]), 14), ("Voovv", "oovv", ([0, 1], [2, 3]), 15)]


def run(ctx, nO, nV, tO, tV, spin, replicated, seed=5):
    if spin:
        Os = tt.IndexSpace(nO, [(0, nO // 2), (nO // 2, nO)], [1, -1])
        Vs = tt.IndexSpace(nV, [(0, nV // 2), (nV // 2, nV)], [1, -1])
        oO = L.IndexSpace(nO, [(0, nO // 2, 1), (nO // 2, nO, -1)])
        oV = L.IndexSpace(nV, [(0, nV // 2, 1), (nV // 2, nV, -1)])
    else:
        Os, Vs, oO, oV = tt.IndexSpace(nO), tt.IndexSpace(nV), L.IndexSpace(nO), L.IndexSpace(nV)
    dims = {"o": tt.TiledIndexSpace(Os, tO), "v": tt.TiledIndexSpace(Vs, tV)}
    odims = {"o": L.tile_fixed(oO, tO), "v": L.tile_fixed(oV, tV)}
    T, dense, keep = {}, {}, [Os, Vs, dims]
    for n, d, sp, tag in INPUTS:
        T[n] = tt.Tensor(ctx, [dims[c] for c in d], spin=sp if spin else None)
        if replicated:
            T[n].set_owner(np.full(T[n].nblocks, tt.TT_REPLICATED, np.int32))
        ot = L.tensor_spin([odims[c] for c in d], *sp) if spin else L.tensor_dense_map([odims[c] for c in d])
        dense[n] = O.dense_masked(ot, S.dense(ot.shape, seed, tag))
        host = O.pack(ot, dense[n])
        if not replicated and ctx.nranks > 1:   # owner-distributed: blocks held elsewhere start as NaN
            for blk in range(T[n].nblocks):
                if T[n].nz[blk] and T[n].owner[blk] not in (ctx.rank, tt.TT_REPLICATED):
                    o = int(T[n].blk_off[blk])
                    ext = [int(dd.offsets[t + 1] - dd.offsets[t]) for dd, t in zip(T[n].dims, np.unravel_index(blk, T[n].grid))]
                    host[o:o + int(np.prod(ext))] = np.nan
        buf = torch.from_numpy(host).cuda()
        T[n].bind(buf)
        keep.append(buf)
    rng = np.random.default_rng(seed)
    eo, ev = rng.uniform(-2, -1, nO), rng.uniform(1, 2, nV)
    args = (T["T1"], T["T2"], T["Vooov"], T["Vvovv"], T["Voovv"])
    _, info = tt.triples_energy(ctx, *args)
    ws = torch.empty(info["ws_elems"], dtype=torch.float64, device="cuda")
    E, info = tt.triples_energy(ctx, *args, torch.from_numpy(eo).cuda(), torch.from_numpy(ev).cuda(), ws)
    orc = (dense["T1"], dense["T2"], dense["Vooov"], dense["Vvovv"], dense["Voovv"], eo, ev)
    return E, info, orc


def main():
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [tt.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    stream = torch.cuda.current_stream().cuda_stream
    ctx = tt.Context(device=local, stream=stream, rank=rank, nranks=world, nccl_id=obj[0])
    ctx1 = tt.Context(device=local, stream=stream)
    ok = True
    for case, repl in (((10, 40, 3, 10, False), True), ((8, 36, 2, 9, True), True), ((8, 36, 2, 9, True), False)):
        # replicated inputs, then owner-distributed ones (round-robin owners, gathered by each rank)
        E, info, orc = run(ctx, *case, replicated=repl)
        E1, info1, _ = run(ctx1, *case, replicated=False)
        units = torch.tensor([info["w_blocks"]], dtype=torch.int64, device="cuda")
        dist.all_reduce(units)
        Eo, _ = TR.energy_by_triple(*orc)
        err = abs(E - Eo) / abs(Eo)
        rel1 = abs(E - E1) / abs(E1)
        good = err <= 1e-11 and rel1 <= 1e-13 and int(units[0]) == info1["w_blocks_total"]
        ok &= good
        if rank == 0:
            print(f"case {case} {'replicated' if repl else 'distributed'}: E={E!r} 1-rank={E1!r} oracle={Eo!r} err={err:.2e} vs1={rel1:.2e} "
                  f"units {int(units[0])}/{info1['w_blocks_total']} {'ok' if good else 'FAIL'}", flush=True)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("MGPU_TRIPLES_CHECK PASS" if int(flag[0]) == 1 else "MGPU_TRIPLES_CHECK FAIL", flush=True)
    ctx.close()
    ctx1.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
