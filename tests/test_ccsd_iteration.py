"""Synthetic CCSD-shaped iteration (configs[3] structure, reading R18): the product driver (Scheduler
over libtt) vs the oracle transcription, on small spin-sparse shapes with several batches of the
implicit Cholesky ladder."""
import numpy as np
import pytest

import synthetic as S
from oracle import layout as L
from oracle import ops as O


def _oracle_tensors(O_, V_, tO, tV, NL, tL):
    from paper_2201_01257_b200.ccsd import TENSORS   # shapes / maps only (the op list is not shared)
    so = L.IndexSpace(O_, [(0, O_ // 2, 1), (O_ // 2, O_, -1)])
    sv = L.IndexSpace(V_, [(0, V_ // 2, 1), (V_ // 2, V_, -1)])
    tis = {"o": L.tile_fixed(so, tO), "v": L.tile_fixed(sv, tV), "L": L.tile_fixed(L.IndexSpace(NL), tL)}
    return {n: (L.tensor_spin([tis[c] for c in cls], up, lo), tag) for n, (cls, (up, lo), tag) in TENSORS.items()}


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(8, 12, 2, 3, 10, 5), (12, 20, 3, 5, 14, 7), (14, 20, 3, 5, 14, 7)])
def test_ccsd_iteration_vs_oracle(shape):
    import torch
    import paper_2201_01257_b200 as tt
    from paper_2201_01257_b200.ccsd import CCSDIteration
    from oracle import ccsd as OC
    O_, V_, tO, tV, NL, tL = shape
    ctx = tt.Context(device=0, stream=torch.cuda.current_stream().cuda_stream)
    it = CCSDIteration(tt, ctx, O_, V_, tO, tV, NL, tL, seed=3, ws_gb=2e-5, nstreams=3)
    nlev, E = it.run()
    got = {n: it.T[n].download() for n in ("R1", "R2", "Wr")}
    ctx.sync()
    ot = _oracle_tensors(*shape)
    D = {n: O.dense_masked(T, S.dense(T.shape, 3, tag)) for n, (T, tag) in ot.items() if tag is not None}
    masks = {n: O.nz_mask(T) for n, (T, tag) in ot.items() if tag is None}
    ref = OC.iterate(D, masks)
    for n in ("R1", "R2", "Wr"):
        r = O.pack(ot[n][0], ref[n])
        assert np.abs(got[n] - r).max() / np.abs(r).max() <= 1e-11, n
    assert abs(E - ref["E"]) <= 1e-12 * abs(ref["E"])
    assert nlev >= 10
