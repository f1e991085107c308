"""Runs the CCSD-shaped term list op by op (direct library calls, no scheduler), synchronising and
printing the per-op time on every rank: locates a slow or hanging operation in multi-GPU runs.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/debug_ccsd_ops.py --O 24 --V 80 --tile 12
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2201_01257_b200 as tt  # noqa: E402
from paper_2201_01257_b200.ccsd import TERMS, CCSDIteration  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--O", type=int, default=24)
    ap.add_argument("--V", type=int, default=80)
    ap.add_argument("--tile", type=int, default=12)
    ap.add_argument("--nl", type=int, default=40)
    ap.add_argument("--ltile", type=int, default=20)
    ap.add_argument("--ws-gb", type=float, default=0.5)
    ap.add_argument("--iters", type=int, default=2)
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
    ctx = tt.Context(device=local, stream=torch.cuda.current_stream().cuda_stream, rank=rank, nranks=world,
                     nccl_id=nid)
    it = CCSDIteration(tt, ctx, a.O, a.V, a.tile, a.tile, a.nl, a.ltile, seed=1, ws_gb=a.ws_gb, nstreams=1)
    T = it.T
    for i in range(a.iters):
        for n, term in enumerate(TERMS):
            t0 = time.time()
            kind = term[0]
            if kind == "add":
                _, out, ol, beta, alpha, x, xl = term
                tt.add(ctx, T[out], ol, beta, alpha, T[x], xl)
            elif kind == "contract":
                _, out, ol, beta, alpha, x, xl, y, yl = term
                tt.contract(ctx, T[out], ol, beta, alpha, T[x], xl, T[y], yl)
            elif kind == "cholesky":
                _, out, ol, beta, alpha, x, xl, y, yl = term
                tt.contract_cholesky(ctx, T[out], ol, beta, alpha, T[x], xl, T[y], yl, it.ws)
            else:
                _, out, ol, beta, alpha, x, xl, y, yl = term
                tt.contract_scalar(ctx, alpha, T[x], xl, T[y], yl)
            torch.cuda.synchronize()
            print(f"rank {rank} iter {i} op {n:2d} {term[:3]} {term[5:]} {1e3 * (time.time() - t0):9.2f} ms",
                  flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
