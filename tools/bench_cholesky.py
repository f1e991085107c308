"""Implicit Cholesky-operand ladder (Eq. cc12) at BASELINE configs[3] scale:
R(a,b,i,j) += V(a,b,c,d) T(c,d,i,j), V(p,q,r,s) = sum_L X(p,r,L)X(q,s,L) - X(p,s,L)X(q,r,L),
O=100 V=800 tile 50 with alpha/beta maps, N_L = 2(O+V) = 1800.  V (1.2 TB as a
spin-packed tensor) is never stored: it is built (DMMA) batch by batch in a workspace and consumed.

    python tools/bench_cholesky.py [--O 100 --V 800 --tile 50 --nl 1800 --ltile 450 --ws-gb 40 --steps 1]

Reports the algorithmic rate (the defined ladder's FLOPs over V's block map / time) and the
executed rate (W build + consume against B - B(c<->d))."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2201_01257_b200 as tt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--O", type=int, default=100)
    ap.add_argument("--V", type=int, default=800)
    ap.add_argument("--tile", type=int, default=50)
    ap.add_argument("--nl", type=int, default=1800)
    ap.add_argument("--ltile", type=int, default=450)
    ap.add_argument("--ws-gb", type=float, default=40.0)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=2)   # >= 2: tt_contract autotunes on the first two calls
    a = ap.parse_args()
    stream = torch.cuda.current_stream()
    ctx = tt.Context(device=0, stream=stream.cuda_stream)
    so = tt.IndexSpace(a.O, [(0, a.O // 2), (a.O // 2, a.O)], [1, -1])
    sv = tt.IndexSpace(a.V, [(0, a.V // 2), (a.V // 2, a.V)], [1, -1])
    sl = tt.IndexSpace(a.nl)
    to, tv, tl = tt.TiledIndexSpace(so, a.tile), tt.TiledIndexSpace(sv, a.tile), tt.TiledIndexSpace(sl, a.ltile)
    R = tt.Tensor(ctx, [tv, tv, to, to], spin=([0, 1], [2, 3]))
    T = tt.Tensor(ctx, [tv, tv, to, to], spin=([0, 1], [2, 3]))
    X = tt.Tensor(ctx, [tv, tv, tl], spin=([0], [1]))
    bufs = []
    for Tn, tag in ((R, 3), (T, 5), (X, 7)):
        b = torch.empty(Tn.packed_elems, dtype=torch.float64, device="cuda")
        Tn.bind(b)
        bufs.append(b)
        tt.fill_synthetic(ctx, Tn, 11, tag)
    ws = torch.empty(int(a.ws_gb * 1e9 / 8), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()

    def step():
        tt.contract_cholesky(ctx, R, "abij", 1.0, 1.0, X, "abcd", T, "cdij", ws)

    t0 = time.time()
    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    plan_s = time.time() - t0
    st = ctx.stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.set_profiling(True)
    ctx.profile_reset()
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    build_ms, nb = ctx.profile("tt_contract_dmma[abcd=")
    cons_ms, nc = ctx.profile("tt_contract_dmma[abij=")
    bm_ms, _ = ctx.profile("tt_add[cholesky Bm]")
    out = {"workload": f"implicit-V ladder O={a.O} V={a.V} tile={a.tile} N_L={a.nl} (L tile {a.ltile}), spin maps",
           "ms_per_step": ms, "algorithmic_flops": st["flops"], "executed_flops": st["aux_flops"],
           "batches": st["work_items"],
           "algorithmic_tflops": st["flops"] / (ms * 1e-3) / 1e12,
           "executed_tflops": st["aux_flops"] / (ms * 1e-3) / 1e12,
           "build_ms": build_ms / a.steps, "consume_ms": cons_ms / a.steps, "bm_prep_ms": bm_ms / a.steps,
           "first_call_s_incl_plans": plan_s, "workspace_gb": a.ws_gb,
           "tensors_gb": {"R": R.packed_elems * 8e-9, "T": T.packed_elems * 8e-9, "X": X.packed_elems * 8e-9}}
    print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
