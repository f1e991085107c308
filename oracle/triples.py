"""Oracle of the perturbative triples correction (T) -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

SURVEY §8(f) NEXT-4; PAPER §4.1.2, P343-413:

* Eq. cc14:   E(T) = sum_{i<j<k, a<b<c} [ <Phi|T2^+ V_N|Phi_ijk^abc> + <Phi|T1^+ V_N|Phi_ijk^abc> ]
                                        * <Phi_ijk^abc|V_N T2|Phi> / (e_i + e_j + e_k - e_a - e_b - e_c)
  For real amplitudes and integrals <Phi|X^+ V_N|Phi_ijk^abc> = <Phi_ijk^abc|V_N X|Phi>, so with
  W = Eq. tensort and V1 = Eq. tensort2:  E(T) = sum (W + V1) * W / D   (reading R28).
* Eq. tensort: W = A + B (Eq. abt), A = the nine terms summed over occupied m, B = the nine terms
  summed over virtual e.  The sixth term is printed "+ v^{ik}_{mc} t^{mj}_{ab}"; the definition
  <Phi_ijk^abc|V_N T2|Phi> is antisymmetric under j<->k, which requires "-" (the third term with j,k
  swapped; P380).  Reading R27: "-" (pinned by a second-quantization evaluation of the definition,
  tests/test_triples.py).
* Eq. tensort2: V1 = nine v^{..}_{..} t^k_c products, as printed.

Storage conventions (the integrals are real, so v^{pq}_{rs} = v^{rs}_{pq} and placement is notation):
  v^{ij}_{ma} = Vooov[i, j, m, a];  v^{ei}_{ab} = Vvovv[e, i, a, b];  v^{ij}_{ab} = Voovv[i, j, a, b];
  t^{ij}_{ab} = T2[a, b, i, j];     t^i_a = T1[a, i];   eps_o[i], eps_v[a] orbital energies.

Plain loops over the restricted (i<j<k, a<b<c) index triples; the per-element sums over m and e are
sequential FP64 in the printed term order (numpy only gathers vectors; the dot products are oracle.c
orc_dot).  Pure Python: for the small parity sizes only.
"""
from __future__ import annotations

import ctypes
import itertools

import numpy as np

from . import _lib


def _dot(x: np.ndarray, y: np.ndarray) -> float:
    xa, ya = _lib.f64(x), _lib.f64(y)
    return float(_lib.lib().orc_dot(len(xa), _lib.ptr(xa, ctypes.c_double), _lib.ptr(ya, ctypes.c_double)))


def w_terms(Vooov, Vvovv, T2, i, j, k, a, b, c):
    """Eq. tensort for one (i,j,k,a,b,c): returns (A, B) of Eq. abt.  Each term is a sequential sum."""
    # A: sum over m of v^{xy}_{m p} t^{m z}_{q r}  (t^{mz}_{qr} = T2[q, r, m, z])
    A = (_dot(Vooov[i, j, :, a], T2[b, c, :, k]) - _dot(Vooov[i, j, :, b], T2[a, c, :, k])
         + _dot(Vooov[i, j, :, c], T2[a, b, :, k]) - _dot(Vooov[i, k, :, a], T2[b, c, :, j])
         + _dot(Vooov[i, k, :, b], T2[a, c, :, j]) - _dot(Vooov[i, k, :, c], T2[a, b, :, j])   # R27
         + _dot(Vooov[j, k, :, a], T2[b, c, :, i]) - _dot(Vooov[j, k, :, b], T2[a, c, :, i])
         + _dot(Vooov[j, k, :, c], T2[a, b, :, i]))
    # B: sum over e of v^{e x}_{p q} t^{y z}_{e r}  (t^{yz}_{er} = T2[e, r, y, z])
    B = (-_dot(Vvovv[:, i, a, b], T2[:, c, j, k]) + _dot(Vvovv[:, i, a, c], T2[:, b, j, k])
         - _dot(Vvovv[:, i, b, c], T2[:, a, j, k]) + _dot(Vvovv[:, j, a, b], T2[:, c, i, k])
         - _dot(Vvovv[:, j, a, c], T2[:, b, i, k]) + _dot(Vvovv[:, j, b, c], T2[:, a, i, k])
         - _dot(Vvovv[:, k, a, b], T2[:, c, i, j]) + _dot(Vvovv[:, k, a, c], T2[:, b, i, j])
         - _dot(Vvovv[:, k, b, c], T2[:, a, i, j]))
    return A, B


def v1_term(Voovv, T1, i, j, k, a, b, c):
    """Eq. tensort2 as printed (t^k_c = T1[c, k])."""
    return (Voovv[i, j, a, b] * T1[c, k] - Voovv[i, j, a, c] * T1[b, k] + Voovv[i, j, b, c] * T1[a, k]
            - Voovv[i, k, a, b] * T1[c, j] + Voovv[i, k, a, c] * T1[b, j] - Voovv[i, k, b, c] * T1[a, j]
            + Voovv[j, k, a, b] * T1[c, i] - Voovv[j, k, a, c] * T1[b, i] + Voovv[j, k, b, c] * T1[a, i])


def energy(T1, T2, Vooov, Vvovv, Voovv, eps_o, eps_v, triples=None):
    """Eq. cc14 over every i<j<k, a<b<c (or the given ((i,j,k),(a,b,c)) list), summed in loop order
    (i<j<k outer, a<b<c inner, both lexicographic).  Returns (E, number of terms)."""
    nO, nV = len(eps_o), len(eps_v)
    E, n = 0.0, 0
    occ = itertools.combinations(range(nO), 3)
    for (i, j, k) in occ:
        for (a, b, c) in itertools.combinations(range(nV), 3):
            A, B = w_terms(Vooov, Vvovv, T2, i, j, k, a, b, c)
            W = A + B
            V1 = v1_term(Voovv, T1, i, j, k, a, b, c)
            D = eps_o[i] + eps_o[j] + eps_o[k] - eps_v[a] - eps_v[b] - eps_v[c]
            E = E + (W + V1) * W / D
            n += 1
    return E, n


def energy_elements(T1, T2, Vooov, Vvovv, Voovv, eps_o, eps_v, elems):
    """The per-element contributions (W + V1) * W / D for a list of (i,j,k,a,b,c) (sampled checks)."""
    out = []
    for (i, j, k, a, b, c) in elems:
        A, B = w_terms(Vooov, Vvovv, T2, i, j, k, a, b, c)
        W = A + B
        V1 = v1_term(Voovv, T1, i, j, k, a, b, c)
        D = eps_o[i] + eps_o[j] + eps_o[k] - eps_v[a] - eps_v[b] - eps_v[c]
        out.append(((W + V1) * W / D, W, V1, D))
    return out


def energy_by_triple(T1, T2, Vooov, Vvovv, Voovv, eps_o, eps_v, max_triples=None):
    """The same Eq. cc14 sum, one occupied triple i<j<k at a time with the 18 terms of Eq. tensort formed
    for all (a,b,c) at once by matrix products (numpy.matmul as the step, P174's contraction of each
    term over m or e), then masked to a<b<c.  Pinned equal to energy() on small sizes; used where the
    element loop is too slow.  ``max_triples`` stops after that many occupied triples (a bounded sample
    for CPU timing).  Returns (E, number of terms).""" 
    nO, nV = len(eps_o), len(eps_v)
    ev = np.asarray(eps_v, dtype=np.float64)
    mask = np.zeros((nV, nV, nV), dtype=bool)
    for a, b, c in itertools.combinations(range(nV), 3):
        mask[a, b, c] = True
    T2o = np.ascontiguousarray(np.transpose(T2, (2, 0, 1, 3)))     # [m][b][c][k]

    def A_term(x, y, z):   # X[a,b,c] = sum_m v^{xy}_{m a} t^{m z}_{b c}
        return np.tensordot(Vooov[x, y], T2o[:, :, :, z], axes=([0], [0]))

    def B_term(x, y, z):   # Y[a,b,c] = sum_e v^{e x}_{a b} t^{y z}_{e c}
        return np.tensordot(Vvovv[:, x], T2[:, :, y, z], axes=([0], [0]))

    E, n = 0.0, 0
    for t, (i, j, k) in enumerate(itertools.combinations(range(nO), 3)):
        if max_triples is not None and t >= max_triples:
            break
        P = lambda X: X - X.transpose(1, 0, 2) + X.transpose(1, 2, 0)  # noqa: E731  X_abc - X_bac + X_cab
        # A: terms 1-3 = P[X_ij,k] over (a|bc): +X(a,b,c) - X(b,a,c) + X(c,a,b)
        A = P(A_term(i, j, k)) - P(A_term(i, k, j)) + P(A_term(j, k, i))
        # B: terms 10-12 = -Y(a,b,c) + Y(a,c,b) - Y(b,c,a) with Y = B_term(i, j, k)
        Q = lambda Y: -Y + Y.transpose(0, 2, 1) - Y.transpose(2, 0, 1)  # noqa: E731
        B = Q(B_term(i, j, k)) - Q(B_term(j, i, k)) + Q(B_term(k, i, j))
        W = A + B
        t1 = lambda x: T1[:, x]  # noqa: E731
        V1 = np.zeros((nV, nV, nV))
        for (x, y, z, s) in ((i, j, k, 1.0), (i, k, j, -1.0), (j, k, i, 1.0)):
            Vxy = Voovv[x, y]
            V1 += s * (np.einsum("ab,c->abc", Vxy, t1(z)) - np.einsum("ac,b->abc", Vxy, t1(z))
                       + np.einsum("bc,a->abc", Vxy, t1(z)))
        D = eps_o[i] + eps_o[j] + eps_o[k] - ev[:, None, None] - ev[None, :, None] - ev[None, None, :]
        with np.errstate(divide="ignore", invalid="ignore"):
            contrib = np.where(mask, (W + V1) * W / np.where(mask, D, 1.0), 0.0)
        E += float(contrib.sum())
        n += int(mask.sum())
    return E, n
