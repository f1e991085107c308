"""Mini-configs of the asynchronous (mbarrier / TMA / cp.async warp-specialised) kernels for
compute-sanitizer (racecheck, synccheck, memcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_mini.py

  * the TMA ladder kernel (tt_contract_tma_kernel): R(abij) += V(abcd) T(cdij), V tile 16 (K = 256);
  * the cp.async warp-specialised kernel on a permuted-output contraction (W-build shape, X(prL) X(qsL));
  * the split-K path and the element kernels (permuted add, scalar);
  * the fused (T) kernel (TMA boxes) on O=6 V=20.
Each result is checked against the CPU oracle so a race that corrupts data also fails the run."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    import torch
    import paper_2201_01257_b200 as tt
    import synthetic as S
    from oracle import ops as O
    from tests.cases import Problem, SpaceSpec, TensorSpec, ccsd_problem, oracle_objects, product_objects
    ctx = tt.Context(device=0, stream=torch.cuda.current_stream().cuda_stream)
    worst = 0.0

    def run(pb, op, alpha=1.0, beta=1.0):
        nonlocal worst
        c, cl, a, al, b, bl = op
        orc = oracle_objects(pb)
        P = product_objects(tt, ctx, pb)
        dense, keep = {}, []
        for name, tag in ((c, 3), (a, 1), (b, 2)):
            dense[name] = O.dense_masked(orc[name], S.dense(orc[name].shape, 1, tag))
            buf = torch.from_numpy(O.pack(orc[name], dense[name])).cuda()
            P[name].bind(buf)
            keep.append(buf)
        tt.contract(ctx, P[c], cl, beta, alpha, P[a], al, P[b], bl)
        got = P[c].download()
        ctx.sync()
        ref = O.pack(orc[c], O.contract(dense[c], cl, dense[a], al, dense[b], bl, alpha, beta, cmask=O.nz_mask(orc[c])))
        err = float(np.abs(got - ref).max() / np.abs(ref).max())
        worst = max(worst, err)
        print(f"{cl}={al}*{bl}: producer {ctx.stats()['producer']} variant {ctx.stats()['kernel_variant']} err {err:.1e}",
              flush=True)

    os.environ["TT_AUTOTUNE"] = "0"
    pb = ccsd_problem(8, 32, 4, 16, False, terms=("ladder",))           # TMA ladder
    run(pb, pb.ops[0])
    pbw = Problem({"V": SpaceSpec(12, tile=6), "L": SpaceSpec(20, tile=10)},
                  {"p": "V", "q": "V", "r": "V", "s": "V", "L": "L"},
                  {"W": TensorSpec("pqrs"), "X": TensorSpec("prL"), "Y": TensorSpec("qsL")},
                  [("W", "pqrs", "X", "prL", "Y", "qsL")])
    run(pbw, pbw.ops[0], beta=0.0)                                       # permuted output (W build)
    pbs = ccsd_problem(4, 40, 2, 10, False, terms=("ring",))             # small output: split-K
    run(pbs, pbs.ops[0])
    # element kernels: permuted add and scalar
    pbe = ccsd_problem(6, 14, 3, 4, True, terms=("ladder",))
    orc = oracle_objects(pbe)
    P = product_objects(tt, ctx, pbe)
    dR = O.dense_masked(orc["R"], S.dense(orc["R"].shape, 2, 3))
    dT = O.dense_masked(orc["T"], S.dense(orc["T"].shape, 2, 5))
    bR, bT = torch.from_numpy(O.pack(orc["R"], dR)).cuda(), torch.from_numpy(O.pack(orc["T"], dT)).cuda()
    P["R"].bind(bR)
    P["T"].bind(bT)
    tt.add(ctx, P["R"], "abij", 1.0, -0.5, P["T"], "baji")
    s = tt.contract_scalar(ctx, 0.25, P["R"], "abij", P["T"], "abij")
    got = P["R"].download()
    ctx.sync()
    refR = O.add(dR, "abij", dT, "baji", -0.5, 1.0, O.nz_mask(orc["R"]))
    err = float(np.abs(got - O.pack(orc["R"], refR)).max())
    serr = abs(s - O.scalar(refR, "abij", dT, "abij", 0.25)) / abs(s)
    print(f"add baji err {err:.1e} scalar err {serr:.1e}", flush=True)
    worst = max(worst, err, serr)
    # (T)
    from tests.test_triples import _gpu_case
    from oracle import triples as TR
    E, info, orc3, _ = _gpu_case(6, 20, 3, 5, False, 3, 1.0)
    Eo, _ = TR.energy(*orc3)
    print(f"(T) E err {abs(E - Eo) / abs(Eo):.1e}", flush=True)
    worst = max(worst, abs(E - Eo) / abs(Eo))
    ctx.close()
    print("SANITIZE_MINI", "PASS" if worst <= 1e-11 else "FAIL", worst, flush=True)
    return 0 if worst <= 1e-11 else 1


if __name__ == "__main__":
    sys.exit(main())
