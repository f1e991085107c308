"""Rank 0's share of the configs[1] ladder at N ranks, timed on ONE GPU (simulated-rank context, inputs
replicated so no exchange is needed): the per-rank kernel time that bench.py --gpus N would see, with
and without the wave tail (run twice, TT_TAIL_SPLIT=1 / 0).

    python tools/probe_tail.py --n 8
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2201_01257_b200 as tt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    group = tt.SimGroup(0, a.n)
    stream = torch.cuda.current_stream()
    ctx = tt.Context(stream=stream.cuda_stream, rank=0, sim=group)
    O, V = tt.IndexSpace(40), tt.IndexSpace(200)
    to, tv = tt.TiledIndexSpace(O, 40), tt.TiledIndexSpace(V, 40)
    R = tt.Tensor(ctx, [tv, tv, to, to])
    Vv = tt.Tensor(ctx, [tv, tv, tv, tv])
    T = tt.Tensor(ctx, [tv, tv, to, to])
    for X in (Vv, T):
        X.set_owner(np.full(X.nblocks, tt.TT_REPLICATED, np.int32))
    tt.partition_split(ctx, R, "abij", Vv, "abcd", T, "cdij", group_dims=(0, 1))
    bufs = []
    for i, X in enumerate((R, Vv, T)):
        b = torch.zeros(X.storage_elems, dtype=torch.float64, device="cuda")
        X.bind(b)
        bufs.append(b)
        tt.fill_synthetic(ctx, X, 1, i + 3)
    for _ in range(3):
        tt.contract(ctx, R, "abij", 1.0, 1.0, Vv, "abcd", T, "cdij")
    st = ctx.stats()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        tt.contract(ctx, R, "abij", 1.0, 1.0, Vv, "abcd", T, "cdij")
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    print(json.dumps({"ranks": a.n, "tail_split": os.environ.get("TT_TAIL_SPLIT", "1"), "ms": ms,
                      "tflops": st["flops"] / (ms * 1e-3) / 1e12, "work_items_main": st["work_items"],
                      "variant": st["kernel_variant"]}), flush=True)
    ctx.close()
    group.close()


if __name__ == "__main__":
    main()
