"""Oracle of the synthetic CCSD iteration -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

Reading R18: the paper gives no CCSD term list (P283-293: "a large number of terms"), so the iteration
is the textbook spin-orbital CCSD residual with the Stanton-Gauss intermediates
(J. F. Stanton, J. Gauss, J. D. Watts, R. J. Bartlett, J. Chem. Phys. 94, 4334 (1991); the form of
the T. D. Crawford / H. F. Schaefer review), evaluated once on seeded synthetic inputs (no molecule, no
convergence).  Every integral is the antisymmetrized <pq||rs> of PAPER Eq. cc12 (P312-318, reading
R19) over the full orbital space o + v:

    <pq||rs> = sum_L X(p,r,L) X(q,s,L) - X(p,s,L) X(q,r,L)

with X given by its four blocks X_oo, X_ov, X_vo, X_vv (reading R30: X(p,r,L) = X(r,p,L) and f
symmetric, as for real orbitals; hermitian_inputs builds them from the seeded raw blocks).  The oracle forms that V
explicitly (oracle.ops.cholesky_v) and transcribes the equations literally, term by term, with the
explicit W_abef intermediate -- independent of the product driver (paper_2201_01257_b200/ccsd.py),
which never forms a >= 3-virtual integral and factorizes those terms through the Cholesky vectors.
The residuals keep the full Fock matrix in F_ae and F_mi (they vanish at convergence; no diagonal
moved to the left-hand side), and E = sum_ia f_ia t_i^a + 1/4 sum_ijab <ij||ab> tau_ij^ab.

Index conventions of the arrays: T1[a,i] = t_i^a, T2[a,b,i,j] = t_ij^ab, fov[i,a] = f_ia.
"""
from __future__ import annotations

import numpy as np

from . import ops as O


def hermitian_inputs(raw: dict) -> dict:
    """The input recipe of the iteration (reading R30), from the seeded raw blocks: real orbitals make
    the Cholesky vectors of (pr|qs) symmetric in (p,r) and the Fock matrix symmetric, so
    X_oo = (R_oo + R_oo^T)/2, X_vv = (R_vv + R_vv^T)/2 (transposing the two orbital indices),
    X_vo = X_ov^T, f_oo = (R + R^T)/2, f_vv = (R + R^T)/2; f_ov, T1, T2 as drawn."""
    D = dict(raw)
    D["Xoo"] = 0.5 * (raw["Xoo"] + raw["Xoo"].transpose(1, 0, 2))
    D["Xvv"] = 0.5 * (raw["Xvv"] + raw["Xvv"].transpose(1, 0, 2))
    D["Xvo"] = raw["Xov"].transpose(1, 0, 2).copy()
    D["foo"] = 0.5 * (raw["foo"] + raw["foo"].T)
    D["fvv"] = 0.5 * (raw["fvv"] + raw["fvv"].T)
    return D


def full_v(D: dict) -> tuple:
    """<pq||rs> over o + v (occupied first) from the X blocks, Eq. cc12 as printed (R19)."""
    nO, nV, NL = D["Xov"].shape
    n = nO + nV
    X = np.zeros((n, n, NL))
    X[:nO, :nO], X[:nO, nO:], X[nO:, :nO], X[nO:, nO:] = D["Xoo"], D["Xov"], D["Xvo"], D["Xvv"]
    return O.cholesky_v(X), slice(0, nO), slice(nO, n)


def iterate(D: dict, masks: dict) -> dict:
    """D: dense inputs foo, fvv, fov, T1, T2, Xoo, Xov, Xvo, Xvv (zero blocks already zero);
    masks: non-zero-block masks of R1 and R2.  Returns dense R1, R2 and the energy E."""
    c, a = O.contract, O.add
    T1, T2, foo, fvv, fov = D["T1"], D["T2"], D["foo"], D["fvv"], D["fov"]
    nV, nO = T1.shape
    V, o, v = full_v(D)
    oooo, ooov, oovv = V[o, o, o, o], V[o, o, o, v], V[o, o, v, v]
    ovov, ovvo, ovoo, oovo = V[o, v, o, v], V[o, v, v, o], V[o, v, o, o], V[o, o, v, o]
    ovvv, vovv, vvvv, vvvo = V[o, v, v, v], V[v, o, v, v], V[v, v, v, v], V[v, v, v, o]
    z = np.zeros
    # tau_ij^ab = t_ij^ab + t_i^a t_j^b - t_i^b t_j^a ; taut = t_ij^ab + 1/2 (t_i^a t_j^b - t_i^b t_j^a)
    tau = c(T2.copy(), "abij", T1, "ai", T1, "bj", 1.0, 1.0)
    tau = c(tau, "abij", T1, "bi", T1, "aj", -1.0, 1.0)
    taut = c(T2.copy(), "abij", T1, "ai", T1, "bj", 0.5, 1.0)
    taut = c(taut, "abij", T1, "bi", T1, "aj", -0.5, 1.0)
    # F_ae = f_ae - 1/2 sum_m f_me t_m^a + sum_mf t_m^f <ma||fe> - 1/2 sum_mnf taut_mn^af <mn||ef>
    Fae = fvv.copy()
    Fae = c(Fae, "ae", fov, "me", T1, "am", -0.5, 1.0)
    Fae = c(Fae, "ae", T1, "fm", ovvv, "mafe", 1.0, 1.0)
    Fae = c(Fae, "ae", taut, "afmn", oovv, "mnef", -0.5, 1.0)
    # F_mi = f_mi + 1/2 sum_e t_i^e f_me + sum_ne t_n^e <mn||ie> + 1/2 sum_nef taut_in^ef <mn||ef>
    Fmi = foo.copy()
    Fmi = c(Fmi, "mi", T1, "ei", fov, "me", 0.5, 1.0)
    Fmi = c(Fmi, "mi", T1, "en", ooov, "mnie", 1.0, 1.0)
    Fmi = c(Fmi, "mi", taut, "efin", oovv, "mnef", 0.5, 1.0)
    # F_me = f_me + sum_nf t_n^f <mn||ef>
    Fme = c(fov.copy(), "me", T1, "fn", oovv, "mnef", 1.0, 1.0)
    # W_mnij = <mn||ij> + P(ij) sum_e t_j^e <mn||ie> + 1/4 sum_ef tau_ij^ef <mn||ef>
    Wmnij = oooo.copy()
    Wmnij = c(Wmnij, "mnij", T1, "ej", ooov, "mnie", 1.0, 1.0)
    Wmnij = c(Wmnij, "mnij", T1, "ei", ooov, "mnje", -1.0, 1.0)
    Wmnij = c(Wmnij, "mnij", tau, "efij", oovv, "mnef", 0.25, 1.0)
    # W_abef = <ab||ef> - P(ab) sum_m t_m^b <am||ef> + 1/4 sum_mn tau_mn^ab <mn||ef>
    Wabef = vvvv.copy()
    Wabef = c(Wabef, "abef", T1, "bm", vovv, "amef", -1.0, 1.0)
    Wabef = c(Wabef, "abef", T1, "am", vovv, "bmef", 1.0, 1.0)
    Wabef = c(Wabef, "abef", tau, "abmn", oovv, "mnef", 0.25, 1.0)
    # W_mbej = <mb||ej> + sum_f t_j^f <mb||ef> - sum_n t_n^b <mn||ej> - sum_nf (1/2 t_jn^fb + t_j^f t_n^b) <mn||ef>
    Wmbej = ovvo.copy()
    Wmbej = c(Wmbej, "mbej", T1, "fj", ovvv, "mbef", 1.0, 1.0)
    Wmbej = c(Wmbej, "mbej", T1, "bn", oovo, "mnej", -1.0, 1.0)
    tq = c(0.5 * T2, "fbjn", T1, "fj", T1, "bn", 1.0, 1.0)
    Wmbej = c(Wmbej, "mbej", tq, "fbjn", oovv, "mnef", -1.0, 1.0)
    # T1 residual
    R1 = a(z((nV, nO)), "ai", fov, "ia", 1.0, 0.0)
    R1 = c(R1, "ai", T1, "ei", Fae, "ae", 1.0, 1.0)
    R1 = c(R1, "ai", T1, "am", Fmi, "mi", -1.0, 1.0)
    R1 = c(R1, "ai", T2, "aeim", Fme, "me", 1.0, 1.0)
    R1 = c(R1, "ai", T1, "fn", ovov, "naif", -1.0, 1.0)
    R1 = c(R1, "ai", T2, "efim", ovvv, "maef", -0.5, 1.0)
    R1 = c(R1, "ai", T2, "aemn", oovo, "nmei", -0.5, 1.0)
    # T2 residual
    R2 = a(z(T2.shape), "abij", oovv, "ijab", 1.0, 0.0)
    # P(ab) sum_e t_ij^ae (F_be - 1/2 sum_m t_m^b F_me)
    Fbe = c(Fae.copy(), "be", T1, "bm", Fme, "me", -0.5, 1.0)
    Zab = c(z(T2.shape), "abij", T2, "aeij", Fbe, "be", 1.0, 0.0)
    # - P(ij) sum_m t_im^ab (F_mj + 1/2 sum_e t_j^e F_me)
    Fmj = c(Fmi.copy(), "mj", T1, "ej", Fme, "me", 0.5, 1.0)
    Zij = c(z(T2.shape), "abij", T2, "abim", Fmj, "mj", -1.0, 0.0)
    # + 1/2 sum_mn tau_mn^ab W_mnij + 1/2 sum_ef tau_ij^ef W_abef
    R2 = c(R2, "abij", tau, "abmn", Wmnij, "mnij", 0.5, 1.0)
    R2 = c(R2, "abij", tau, "efij", Wabef, "abef", 0.5, 1.0)
    # + P(ij) P(ab) sum_me (t_im^ae W_mbej - t_i^e t_m^a <mb||ej>)
    Zr = c(z(T2.shape), "abij", T2, "aeim", Wmbej, "mbej", 1.0, 0.0)
    tt1 = c(z((nV, nV, nO, nO)), "eaim", T1, "ei", T1, "am", 1.0, 0.0)     # t_i^e t_m^a
    Zr = c(Zr, "abij", tt1, "eaim", ovvo, "mbej", -1.0, 1.0)
    # + P(ij) sum_e t_i^e <ab||ej> ; - P(ab) sum_m t_m^a <mb||ij>
    Zij = c(Zij, "abij", T1, "ei", vvvo, "abej", 1.0, 1.0)
    Zab = c(Zab, "abij", T1, "am", ovoo, "mbij", -1.0, 1.0)
    for lbl, sgn in (("abij", 1.0), ("baij", -1.0)):
        R2 = a(R2, "abij", Zab, lbl, sgn, 1.0)
    for lbl, sgn in (("abij", 1.0), ("abji", -1.0)):
        R2 = a(R2, "abij", Zij, lbl, sgn, 1.0)
    for lbl, sgn in (("abij", 1.0), ("baij", -1.0), ("abji", -1.0), ("baji", 1.0)):
        R2 = a(R2, "abij", Zr, lbl, sgn, 1.0)
    R1 = np.where(masks["R1"].astype(bool), R1, 0.0)
    R2 = np.where(masks["R2"].astype(bool), R2, 0.0)
    E = O.scalar(fov, "ia", T1, "ai", 1.0) + O.scalar(oovv, "ijab", tau, "abij", 0.25)
    return {"R1": R1, "R2": R2, "E": E}
