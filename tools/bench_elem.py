"""HBM-bound element operations (SURVEY §8(a) A8 add, A9 set, A10 scalar) on cfg3-sized tensors.

    python tools/bench_elem.py [--steps K]

R, Rt, T2 are (V,V,O,O)-shaped spin-sparse doubles amplitudes of config 3 (O=60, V=400, tO=30, tV=40;
1.728 GB each packed).  Reports kernel time (libtt CUDA events) and achieved GB/s of algorithmic
bytes against the measured HBM copy bandwidth (MEASURED_PEAKS.json hbm_gbs)."""
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
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = peaks["hbm_gbs"]
    ctx = tt.Context(device=0, stream=torch.cuda.current_stream().cuda_stream)
    so = tt.IndexSpace(60, [(0, 30), (30, 60)], [1, -1])
    sv = tt.IndexSpace(400, [(0, 200), (200, 400)], [1, -1])
    to, tv = tt.TiledIndexSpace(so, 30), tt.TiledIndexSpace(sv, 40)
    R = tt.Tensor(ctx, [tv, tv, to, to], spin=([0, 1], [2, 3]))
    Rt = tt.Tensor(ctx, [to, to, tv, tv], spin=([0, 1], [2, 3]))
    T2 = tt.Tensor(ctx, [tv, tv, to, to], spin=([0, 1], [2, 3]))
    T2p = tt.Tensor(ctx, [tv, to, tv, to], spin=([0, 2], [1, 3]))
    bufs = []
    for i, T in enumerate((R, Rt, T2, T2p)):
        b = torch.empty(T.packed_elems, dtype=torch.float64, device="cuda")
        T.bind(b)
        bufs.append(b)
        tt.fill_synthetic(ctx, T, 5, i + 1)
    n = R.packed_elems
    ops = [
        ("set R = 1", lambda: tt.set_(ctx, R, 1.0), "tt_set", 8 * n),
        ("add R(abij) = R + T2(abij) (identity)", lambda: tt.add(ctx, R, "abij", 1.0, 0.5, T2, "abij"), "tt_add", 24 * n),
        ("add R(abij) = R + Rt(ijab) (transpose)", lambda: tt.add(ctx, R, "abij", 1.0, 0.5, Rt, "ijab"), "tt_add", 24 * n),
        ("add R(abij) = T2p(aibj) (beta=0, 4-d permutation)", lambda: tt.add(ctx, R, "abij", 0.0, 1.0, T2p, "aibj"), "tt_add", 16 * n),
        ("add R(abij) = R - T2(baij) (antisymmetrizer, rows of 900)", lambda: tt.add(ctx, R, "abij", 1.0, -1.0, T2, "baij"), "tt_add", 24 * n),
        ("scalar T2(abij) . R(abij)", lambda: tt.contract_scalar(ctx, 0.25, T2, "abij", R, "abij"), "tt_scalar_partials", 16 * n),
        ("scalar Rt(ijab) . R(abij) (permuted)", lambda: tt.contract_scalar(ctx, 0.25, Rt, "ijab", R, "abij"), "tt_scalar_partials", 16 * n),
        ("scalar T2p(aibj) . R(abij) (4-d permutation)", lambda: tt.contract_scalar(ctx, 0.25, T2p, "aibj", R, "abij"), "tt_scalar_partials", 16 * n),
    ]
    out = []
    for name, fn, kern, nbytes in ops:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ctx.set_profiling(True)
        ctx.profile_reset()
        for _ in range(args.steps):
            fn()
        ms, k = ctx.profile(kern)
        ctx.set_profiling(False)
        avg = ms / max(k, 1)
        gbs = nbytes / (avg * 1e-3) / 1e9
        out.append({"op": name, "kernel": kern, "kernel_ms": avg, "bytes": nbytes, "GB/s": gbs, "frac_hbm": gbs / hbm})
        print(json.dumps(out[-1]), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
