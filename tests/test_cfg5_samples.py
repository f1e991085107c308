"""BASELINE configs[4] parity on the committed GPU runs: tools/bench_cfg5.py --samples-out wrote
sampled R(a,b,i,j) elements of the large implicit-Cholesky ladder (O=150, V up to 1200, tile 64,
N_L = 2(O+V), 1-4 B200s) to profiles/r01_cfg5_samples_*.json; here the oracle recomputes each one
from the seeded inputs -- one (a,b) row of Eq. cc12 (oracle.ops.cholesky_v_row, two products over
L) against T(:,:,i,j) -- and the GPU values must agree normwise within 1e-11 (SURVEY §8(c) step 6:
samples grouped by (a,b) row).  Zero blocks (spin rule R7) are masked on the oracle side."""
import glob
import json
import os

import numpy as np
import pytest

import synthetic as S
from oracle import ops as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FILES = sorted(glob.glob(os.path.join(ROOT, "profiles", "*cfg5_samples*.json")))


def _spin(x, n):
    return np.where(np.asarray(x) < n // 2, 1, -1)


@pytest.mark.skipif(not FILES, reason="no committed configs[4] sample file")
@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f) for f in FILES])
def test_cfg5_samples_vs_oracle(path):
    rec = json.load(open(path))
    Oc, Vc, NL, seed, alpha = rec["O"], rec["V"], rec["NL"], rec["seed"], rec["alpha"]
    tags = rec["tags"]
    smp = np.array(rec["samples"], dtype=np.float64)
    assert len(smp) >= 12
    rows = sorted({(int(a), int(b)) for a, b in smp[:, :2]})
    r = np.arange(Vc)
    sv = _spin(r, Vc)
    ref, got = [], []
    for a, b in rows:
        # X(p, r, L) rows p = a, b, zero unless spin p == spin r (X's map, R7)
        L = np.arange(NL)
        xr = []
        for p in (a, b):
            idx = np.stack(np.broadcast_arrays(np.full((Vc, NL), p), r[:, None], L[None, :]), axis=-1)
            vals = S.values(seed, tags["X"], S.linear_index((Vc, Vc, NL), idx))
            xr.append(np.where((sv == _spin(p, Vc))[:, None], vals, 0.0))
        vrow = O.cholesky_v_row(xr[0], xr[1])
        for s in smp[(smp[:, 0] == a) & (smp[:, 1] == b)]:
            i, j = int(s[2]), int(s[3])
            idx = np.stack(np.broadcast_arrays(r[:, None], r[None, :], np.full((Vc, Vc), i), np.full((Vc, Vc), j)), axis=-1)
            t = S.values(seed, tags["T"], S.linear_index((Vc, Vc, Oc, Oc), idx))
            conserve = (sv[:, None] + sv[None, :]) == (_spin(i, Oc) + _spin(j, Oc))
            ref.append(O.ladder_sample(vrow, np.where(conserve, t, 0.0), alpha))
            got.append(s[4])
    ref, got = np.array(ref), np.array(got)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err <= 1e-11, err
