"""Multi-GPU parity check of the synthetic CCSD-shaped iteration (run under torchrun, NCCL).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port 29513 tests/mgpu_ccsd_check.py

CCSDIteration distributes its tensors (replicated inputs and small intermediates, row-split R2 / Wr /
Z / Q / Q' / K3); every rank runs the scheduler; the owned parts of R2 are assembled on rank 0 (sum of
the owned elements: each element has exactly one owner, replicated blocks counted from rank 0) and
compared with the oracle transcription (normwise 1e-11), R1 and the energy too."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2201_01257_b200 as tt  # noqa: E402
from oracle import ops as O  # noqa: E402
from tests.test_ccsd_iteration import oracle_reference  # noqa: E402


def owned(T, got, rank):
    """Packed-layout copy of the storage buffer ``got`` with only the elements this rank owns
    (replicated blocks: rank 0); works for compact storage (storage_off) and the full layout."""
    mine = np.zeros(T.packed_elems)
    for blk in range(T.nblocks):
        if not T.nz[blk]:
            continue
        o, so = T.blk_off[blk], T.storage_off[blk]
        ext = [d.offsets[t + 1] - d.offsets[t] for d, t in zip(T.dims, np.unravel_index(blk, T.grid))]
        n = int(np.prod(ext))
        if T.owner[blk] == rank or (T.owner[blk] == tt.TT_REPLICATED and rank == 0):
            mine[o:o + n] = got[so:so + n]
        inner = n // int(ext[0])
        for (bb, lo, hi, ow) in T.parts:
            if bb == blk and ow == rank:
                mine[o + lo * inner:o + hi * inner] = got[so + lo * inner:so + hi * inner]
    return mine


def main():
    from paper_2201_01257_b200.ccsd import CCSDIteration
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [tt.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    stream = torch.cuda.current_stream().cuda_stream
    ctx = tt.Context(device=local, stream=stream, rank=rank, nranks=world, nccl_id=obj[0])
    ok = True
    for shape in ((12, 20, 3, 5, 14, 7), (16, 40, 4, 6, 24, 10)):
        it = CCSDIteration(tt, ctx, *shape, seed=3, ws_gb=2e-3, nstreams=3)
        for rep in range(2):      # the second run replays the cached plans
            nlev, E = it.run()
            res = {}
            for n in ("R1", "R2"):
                g = it.T[n].download()
                ctx.sync()
                t = torch.from_numpy(owned(it.T[n], g, rank)).cuda()
                dist.all_reduce(t)
                res[n] = t.cpu().numpy()
            if rank == 0:
                if rep == 0:
                    ot, ref = oracle_reference(shape, 3)
                errs = {}
                for n in ("R1", "R2"):
                    r = O.pack(ot[n][0], ref[n])
                    errs[n] = float(np.abs(res[n] - r).max() / np.abs(r).max())
                eE = abs(E - ref["E"]) / abs(ref["E"])
                good = all(e <= 1e-11 for e in errs.values()) and eE <= 1e-11
                ok &= good
                print(f"world {world} shape {shape} run {rep}: levels {nlev} errors {errs} energy {eE:.2e} "
                      f"{'ok' if good else 'BAD'}", flush=True)
    if rank == 0:
        print("MGPU_CCSD_CHECK", "PASS" if ok else "FAIL", flush=True)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
