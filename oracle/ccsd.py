"""Oracle of the synthetic CCSD-shaped iteration -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

Reading R18: the paper gives no CCSD term list (P283-293); the iteration is a frozen CCSD-shaped list
(tau-based ladder with the Cholesky-factored V of Eq. cc12, Woooo / Wovvo / Fvv / Foo / Fov
intermediates, P(ab)/P(ij) antisymmetrizers, energy 1/4 <ij||ab> tau).  This module transcribes it
independently of the product driver (paper_2201_01257_b200/ccsd.py), term by term, with the oracle's
dense FP64 operations; the GPU test compares the two results.
"""
from __future__ import annotations

import numpy as np

from . import ops as O


def iterate(D: dict, masks: dict) -> dict:
    """D: dense inputs foo, fvv, T1, T2, Voovv, Voooo, Wr, X (zero blocks already zero);
    masks: non-zero-block masks of the outputs tau, Wo, Fv, Fo, Fov, Z, R2, R1.
    Returns the dense R1, R2, Wr (updated in place by the iteration) and the energy E."""
    c, a, s = O.contract, O.add, O.scalar
    m = masks
    T1, T2, Vo, X = D["T1"], D["T2"], D["Voovv"], D["X"]
    # tau_ij^ab = t_ij^ab + t_i^a t_j^b - t_i^b t_j^a
    tau = a(np.zeros_like(T2), "abij", T2, "abij", 1.0, 0.0, m["tau"])
    tau = c(tau, "abij", T1, "ai", T1, "bj", 1.0, 1.0, m["tau"])
    tau = c(tau, "abij", T1, "bi", T1, "aj", -1.0, 1.0, m["tau"])
    # Woooo
    Wo = a(np.zeros_like(D["Voooo"]), "klij", D["Voooo"], "klij", 1.0, 0.0, m["Wo"])
    Wo = c(Wo, "klij", Vo, "cdkl", tau, "cdij", 0.25, 1.0, m["Wo"])
    # Wovvo (in place on the input)
    Wr = c(D["Wr"], "kbcj", T2, "dblj", Vo, "cdkl", -0.5, 1.0, None)
    # Fvv, Foo, Fov
    Fv = a(np.zeros_like(D["fvv"]), "ae", D["fvv"], "ae", 1.0, 0.0, m["Fv"])
    Fv = c(Fv, "ae", T2, "afmn", Vo, "efmn", -0.5, 1.0, m["Fv"])
    Fo = a(np.zeros_like(D["foo"]), "mi", D["foo"], "mi", 1.0, 0.0, m["Fo"])
    Fo = c(Fo, "mi", Vo, "efmn", T2, "efin", 0.5, 1.0, m["Fo"])
    nO, nV = D["foo"].shape[0], D["fvv"].shape[0]
    Fov = c(np.zeros((nO, nV)), "me", Vo, "efmn", T1, "fn", 1.0, 0.0, m["Fov"])
    # doubles residual
    R2 = a(np.zeros_like(T2), "abij", Vo, "abij", 1.0, 0.0, m["R2"])
    V = O.cholesky_v(X)                                   # Eq. cc12, formed explicitly here
    R2 = c(R2, "abij", V, "abcd", tau, "cdij", 0.5, 1.0, m["R2"])
    R2 = c(R2, "abij", tau, "abkl", Wo, "klij", 0.5, 1.0, m["R2"])
    Z = c(np.zeros_like(T2), "abij", T2, "acik", Wr, "kbcj", 1.0, 0.0, m["Z"])
    for lbl, sgn in (("abij", 1.0), ("baij", -1.0), ("abji", -1.0), ("baji", 1.0)):     # P(ab) P(ij)
        R2 = a(R2, "abij", Z, lbl, sgn, 1.0, m["R2"])
    Z = c(np.zeros_like(T2), "abij", T2, "aeij", Fv, "be", 1.0, 0.0, m["Z"])
    for lbl, sgn in (("abij", 1.0), ("baij", -1.0)):                                      # P(ab)
        R2 = a(R2, "abij", Z, lbl, sgn, 1.0, m["R2"])
    Z = c(np.zeros_like(T2), "abij", T2, "abim", Fo, "mj", 1.0, 0.0, m["Z"])
    for lbl, sgn in (("abij", -1.0), ("abji", 1.0)):                                      # -P(ij)
        R2 = a(R2, "abij", Z, lbl, sgn, 1.0, m["R2"])
    # singles residual
    R1 = c(np.zeros_like(T1), "ai", Fv, "ae", T1, "ei", 1.0, 0.0, m["R1"])
    R1 = c(R1, "ai", T1, "am", Fo, "mi", -1.0, 1.0, m["R1"])
    R1 = c(R1, "ai", T2, "aeim", Fov, "me", 1.0, 1.0, m["R1"])
    E = s(Vo, "abij", tau, "abij", 0.25)
    return {"R1": R1, "R2": R2, "Wr": Wr, "E": E}
