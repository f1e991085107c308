"""Launch-bound small contractions (BASELINE configs[0]: ring C(a,b,i,j) += A(a,c,i,k) B(c,b,k,j),
O=4 V=8 tile 4): wall time per contraction through the immediate ABI call vs a CUDA graph of the
scheduler queue (tt_sched_capture / tt_sched_replay), host loop included."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2201_01257_b200 as tt  # noqa: E402


def main():
    if "--variants" in sys.argv:   # per kernel variant (TT_FORCE_VARIANT), each in a fresh process
        import subprocess
        for v in range(6):
            env = dict(os.environ, TT_FORCE_VARIANT=str(v))
            out = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True).stdout
            print(json.dumps({"variant": v, **json.loads(out.strip().splitlines()[-1])}), flush=True)
        return
    stream = torch.cuda.current_stream()
    ctx = tt.Context(device=0, stream=stream.cuda_stream)
    so, sv = tt.IndexSpace(4), tt.IndexSpace(8)
    to, tv = tt.TiledIndexSpace(so, 4), tt.TiledIndexSpace(sv, 4)
    C, A, B = (tt.Tensor(ctx, [tv, tv, to, to]), tt.Tensor(ctx, [tv, tv, to, to]), tt.Tensor(ctx, [tv, tv, to, to]))
    bufs = []
    for T, tag in ((C, 3), (A, 1), (B, 2)):
        b = torch.empty(T.packed_elems, dtype=torch.float64, device="cuda")
        T.bind(b)
        bufs.append(b)
        tt.fill_synthetic(ctx, T, 1, tag)
    n = 200
    for _ in range(10):
        tt.contract(ctx, C, "abij", 1.0, 1e-3, A, "acik", B, "cbkj")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        tt.contract(ctx, C, "abij", 1.0, 1e-3, A, "acik", B, "cbkj")
    torch.cuda.synchronize()
    imm = (time.perf_counter() - t0) / n * 1e6
    k = 20
    s = tt.Scheduler(ctx, nstreams=1)
    for _ in range(k):
        s.contract(C, "abij", 1.0, 1e-3, A, "acik", B, "cbkj")
    s.capture()
    s.replay()
    torch.cuda.synchronize()
    reps = 50
    t0 = time.perf_counter()
    for _ in range(reps):
        s.replay()
    torch.cuda.synchronize()
    gr = (time.perf_counter() - t0) / (reps * k) * 1e6
    ctx.set_profiling(True)
    ctx.profile_reset()
    for _ in range(n):
        tt.contract(ctx, C, "abij", 1.0, 1e-3, A, "acik", B, "cbkj")
    kms, kn = ctx.profile("tt_contract_dmma")
    ctx.set_profiling(False)
    print(json.dumps({"workload": "configs[0] ring O=4 V=8 tile 4 (65536 FLOPs)", "immediate_us_per_contraction": imm,
                      "graph_us_per_contraction": gr, "contractions_per_graph": k,
                      "kernel_us_events": kms / max(kn, 1) * 1e3, "variant": ctx.stats()["kernel_variant"]}))


if __name__ == "__main__":
    main()
