"""Host recheck of full-size sampled outputs written by the GPU tools (run on the GPU box after the
tool; test infrastructure: calls only oracle/).  Adds a "check" section to the samples file.

    python tests/full_samples_check.py ccsd  <file>   # tools/bench_ccsd.py --samples-out (configs[3])
    python tests/full_samples_check.py cfg5  <file>   # tools/bench_cfg5.py --samples-out (configs[4])

ccsd: every sampled R1 / R2 element by oracle/ccsd_sample.py (element-wise form of the literal CCSD
oracle, pinned to it on mini shapes).  cfg5: every sampled ladder element R(a,b,i,j) = alpha * sum_cd
v(a,b,c,d) T(c,d,i,j) with the row v(a,b,:,:) of Eq. cc12 (oracle.ops.cholesky_v_row) from the seeded
X, T(:,:,i,j) from the seeded T (spin maps R7).  Norm (reading R13): the largest |reference| over the
samples."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synthetic as S  # noqa: E402
from oracle import ops as O  # noqa: E402


def _spin(x, n):
    return np.where(np.asarray(x) < n // 2, 1, -1)


def cfg5_reference(rec, rows_limit=None):
    """Reference values of the samples of a bench_cfg5 record (grouped by (a,b) row)."""
    Oc, Vc, NL, seed, alpha, tags = rec["O"], rec["V"], rec["NL"], rec["seed"], rec["alpha"], rec["tags"]
    smp = np.array(rec["samples"], dtype=np.float64)
    rows = []
    for a, b in smp[:, :2].astype(int):
        if (a, b) not in rows:
            rows.append((a, b))
    if rows_limit:
        rows = rows[:rows_limit]
    r = np.arange(Vc)
    sv = _spin(r, Vc)
    L = np.arange(NL)
    ref, got = [], []
    for a, b in rows:
        xr = []
        for p in (a, b):   # X(p, r, L), zero unless spin p == spin r (X's map, R7)
            idx = np.stack(np.broadcast_arrays(np.full((Vc, NL), p), r[:, None], L[None, :]), axis=-1)
            vals = S.values(seed, tags["X"], S.linear_index((Vc, Vc, NL), idx))
            xr.append(np.where((sv == _spin(p, Vc))[:, None], vals, 0.0))
        vrow = O.cholesky_v_row(xr[0], xr[1])
        for s in smp[(smp[:, 0] == a) & (smp[:, 1] == b)]:
            i, j = int(s[2]), int(s[3])
            idx = np.stack(np.broadcast_arrays(r[:, None], r[None, :], np.full((Vc, Vc), i), np.full((Vc, Vc), j)),
                           axis=-1)
            t = S.values(seed, tags["T"], S.linear_index((Vc, Vc, Oc, Oc), idx))
            conserve = (sv[:, None] + sv[None, :]) == (_spin(i, Oc) + _spin(j, Oc))
            ref.append(O.ladder_sample(vrow, np.where(conserve, t, 0.0), alpha))
            got.append(s[4])
    return np.array(ref), np.array(got)


def main():
    kind, path = sys.argv[1], sys.argv[2]
    rec = json.load(open(path))
    t0 = time.time()
    if kind == "ccsd":
        from oracle.ccsd_sample import Inputs, Sampler
        c = rec["config"]
        sm = Sampler(Inputs(c["O"], c["V"], c["N_L"], c["seed"]))
        ref2 = [sm.r2(*map(int, p[:4])) for p in rec["r2"]]
        ref1 = [sm.r1(*map(int, p[:2])) for p in rec["r1"]]
        g2, g1 = np.array([p[4] for p in rec["r2"]]), np.array([p[2] for p in rec["r1"]])
        rec["check"] = {"r2_ref": ref2, "r1_ref": ref1, "seconds": time.time() - t0,
                        "r2_normwise": float(np.abs(g2 - ref2).max() / np.abs(ref2).max()),
                        "r1_normwise": float(np.abs(g1 - ref1).max() / np.abs(ref1).max()),
                        "how": "tests/full_samples_check.py: oracle/ccsd_sample.py on the host cores"}
        err = max(rec["check"]["r2_normwise"], rec["check"]["r1_normwise"])
    else:
        ref, got = cfg5_reference(rec)
        err = float(np.abs(got - ref).max() / np.abs(ref).max())
        rec["check"] = {"normwise": err, "samples": int(len(ref)), "seconds": time.time() - t0,
                        "how": "tests/full_samples_check.py: oracle.ops.cholesky_v_row + ladder_sample"}
    json.dump(rec, open(path, "w"), indent=1)
    print("FULL_SAMPLES_CHECK", kind, os.path.basename(path), "PASS" if err <= 1e-11 else "FAIL", err, flush=True)
    return 0 if err <= 1e-11 else 1


if __name__ == "__main__":
    sys.exit(main())
