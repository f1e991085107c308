"""NEXT-3 measurement: the cc9 term R(a,b,i,j) += 1/4 v(e,f,m,n) t(e,f,i,j) t(a,b,m,n) (PAPER Eqs. cc9-cc11)
through tt_contract3 at configs[2] sizes (O=60, V=400, tiles 30 / 40, alpha/beta maps or dense).

    python tools/bench_contract3.py [--O 60 --V 400 --tO 30 --tV 40 --dense]

Reports the pairing the library chose, the FLOPs it executes (both binary contractions), the naive
multiply-adds of the unfactorized loop (the n_o^4 n_u^4 class of P299) and the device time per call
(CUDA events, after warm-up; inputs seeded synthetic, resident in HBM)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2201_01257_b200 as tt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--O", type=int, default=60)
    ap.add_argument("--V", type=int, default=400)
    ap.add_argument("--tO", type=int, default=30)
    ap.add_argument("--tV", type=int, default=40)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    stream = torch.cuda.current_stream()
    ctx = tt.Context(device=0, stream=stream.cuda_stream)
    if a.dense:
        O, V = tt.IndexSpace(a.O), tt.IndexSpace(a.V)
    else:
        O = tt.IndexSpace(a.O, [(0, a.O // 2), (a.O // 2, a.O)], [1, -1])
        V = tt.IndexSpace(a.V, [(0, a.V // 2), (a.V // 2, a.V)], [1, -1])
    to, tv = tt.TiledIndexSpace(O, a.tO), tt.TiledIndexSpace(V, a.tV)
    sp = None if a.dense else ([0, 1], [2, 3])
    R = tt.Tensor(ctx, [tv, tv, to, to], spin=sp)
    v = tt.Tensor(ctx, [tv, tv, to, to], spin=sp)
    t = tt.Tensor(ctx, [tv, tv, to, to], spin=sp)
    bufs = []
    for X, tag in ((R, 3), (v, 6), (t, 5)):
        b = torch.empty(X.packed_elems, dtype=torch.float64, device="cuda")
        X.bind(b)
        tt.fill_synthetic(ctx, X, 1, tag)
        bufs.append(b)
    args = (ctx, R, "abij", 1.0, 0.25, v, "efmn", t, "efij", t, "abmn")
    plan = tt.contract3(*args)
    ws = torch.empty(plan["ws_elems"], dtype=torch.float64, device="cuda")
    for _ in range(a.warmup):
        tt.contract3(*args, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        tt.contract3(*args, ws)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    st = ctx.stats()
    f = plan["flops"][plan["pair"]]
    print(json.dumps({"workload": f"cc9 R(abij) += 1/4 v(efmn) t(efij) t(abmn), O={a.O} V={a.V} tO={a.tO} tV={a.tV} "
                                  f"{'dense' if a.dense else 'alpha/beta maps'}",
                      "pair": ["(A*B)*D", "(A*D)*B", "(B*D)*A"][plan["pair"]], "intermediate": plan["i_lbl"],
                      "factorized_flops": f, "flops_of_pairings": plan["flops"], "naive_macs": plan["naive_macs"],
                      "naive_over_factorized_macs": plan["naive_macs"] / (f / 2) if f > 0 else None,
                      "ms_per_call": ms, "tflops": f / ms / 1e9, "pct_fp64_peak": f / ms / 1e9 / 37.1 * 100,
                      "stats_flops": st["flops"], "workspace_gb": plan["ws_elems"] * 8e-9}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
