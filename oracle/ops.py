"""Oracle operations over dense global arrays -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

The method reaches exactly (up to rounding order) the plain definition, so the oracle IS the plain
definition:

* contraction (P174, rule 7):  for every element x of every NON-ZERO C block
      C[x] <- beta*C[x] + alpha * sum_{y over contracted global index tuples} A[x_A, y_A] * B[x_B, y_B]
  zero blocks of A and B read as 0 (S216); zero C blocks stay absent (reading R8).
* addition (P173, rule 6):     C[x] <- beta*C[x] + alpha*A[pi(x)]   on non-zero C blocks
* set (P172, rule 5):          C[x] <- alpha                        on non-zero C blocks
* scalar contraction (order-0 result, P534-536 energy as a sum of contributions):
      s = alpha * sum_x A[x_A] * B[x_B]

The loops of contract/add/set/scalar are in oracle.c (sequential FP64 sums, reading R12); there numpy
only moves data (transpose/copy = memory order) and builds masks.  Library reductions appear only in
the sampled checks for sizes the loops cannot reach, each named in its docstring as a library
primitive and pinned in tests/test_oracle_pins.py: cholesky_v_row (BLAS matrix products over L),
ladder_sample (numpy.sum), freivalds (numpy.einsum).
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .layout import Tensor, analyse_labels


# ----------------------------------------------------------------------------- packed <-> dense

def unpack(T: Tensor, packed: np.ndarray) -> np.ndarray:
    """Packed non-zero blocks -> dense global array (zero blocks = 0), own addressing:
    block id -> tile origin -> global slice (P111, reading R9/R10)."""
    D = np.zeros(T.shape, dtype=np.float64)
    offs = T.blk_off()
    for b in range(T.nblocks()):
        if offs[b] < 0:
            continue
        o, e = T.block_origin(b), T.block_extents(b)
        vol = T.block_volume(b)
        sl = tuple(slice(oo, oo + ee) for oo, ee in zip(o, e))
        D[sl] = packed[offs[b]:offs[b] + vol].reshape(e)
    return D


def pack(T: Tensor, D: np.ndarray) -> np.ndarray:
    """Dense global array -> packed storage of the non-zero blocks (padding = 0)."""
    P = np.zeros(T.packed_elems(), dtype=np.float64)
    offs = T.blk_off()
    for b in range(T.nblocks()):
        if offs[b] < 0:
            continue
        o, e = T.block_origin(b), T.block_extents(b)
        sl = tuple(slice(oo, oo + ee) for oo, ee in zip(o, e))
        P[offs[b]:offs[b] + T.block_volume(b)] = D[sl].reshape(-1)
    return P


def nz_mask(T: Tensor) -> np.ndarray:
    """Dense u8 mask over T's global shape: 1 where the element lies in a non-zero block."""
    M = np.zeros(T.shape, dtype=np.uint8)
    for b in range(T.nblocks()):
        if T.nz[b]:
            o, e = T.block_origin(b), T.block_extents(b)
            M[tuple(slice(oo, oo + ee) for oo, ee in zip(o, e))] = 1
    return M


def dense_masked(T: Tensor, D: np.ndarray) -> np.ndarray:
    """Zero blocks read as zeros (S216): D with every zero block cleared."""
    return np.where(nz_mask(T).astype(bool), D, 0.0)


# ----------------------------------------------------------------------------- contraction

def _strides(shape):
    s, acc = [], 1
    for n in reversed(shape):
        s.append(acc)
        acc *= int(n)
    return list(reversed(s))


def contract_naive(C: np.ndarray, c_lbl: str, A: np.ndarray, a_lbl: str, B: np.ndarray, b_lbl: str,
                   alpha: float, beta: float, cmask: Optional[np.ndarray] = None) -> np.ndarray:
    """Strided nested loops (oracle.c orc_contract_naive).  Returns a new C array."""
    L = analyse_labels(c_lbl, a_lbl, b_lbl)
    ext = {}
    for arr, lbl in ((C, c_lbl), (A, a_lbl), (B, b_lbl)):
        for n, x in zip(arr.shape, lbl):
            if ext.setdefault(x, n) != n:
                raise ValueError(f"extent mismatch on label {x}")
    sc, sa, sb = _strides(C.shape), _strides(A.shape), _strides(B.shape)
    ext_f = _lib.i64([ext[x] for x in c_lbl])
    sfc = _lib.i64([sc[c_lbl.index(x)] for x in c_lbl])
    sfa = _lib.i64([sa[a_lbl.index(x)] if x in a_lbl else 0 for x in c_lbl])
    sfb = _lib.i64([sb[b_lbl.index(x)] if x in b_lbl else 0 for x in c_lbl])
    ext_k = _lib.i64([ext[x] for x in L.con] or [1])
    ska = _lib.i64([sa[a_lbl.index(x)] for x in L.con] or [0])
    skb = _lib.i64([sb[b_lbl.index(x)] for x in L.con] or [0])
    Co = _lib.f64(C).copy()
    Ao, Bo = _lib.f64(A), _lib.f64(B)
    m = None if cmask is None else np.ascontiguousarray(cmask, dtype=np.uint8)
    lib = _lib.lib()
    lib.orc_contract_naive(len(c_lbl), _lib.ptr(ext_f, ctypes.c_int64), _lib.ptr(sfc, ctypes.c_int64),
                           _lib.ptr(sfa, ctypes.c_int64), _lib.ptr(sfb, ctypes.c_int64), len(L.con),
                           _lib.ptr(ext_k, ctypes.c_int64), _lib.ptr(ska, ctypes.c_int64),
                           _lib.ptr(skb, ctypes.c_int64), _lib.ptr(Co, ctypes.c_double),
                           _lib.ptr(Ao, ctypes.c_double), _lib.ptr(Bo, ctypes.c_double),
                           None if m is None else _lib.ptr(m, ctypes.c_uint8), float(alpha), float(beta))
    return Co


def contract(C: np.ndarray, c_lbl: str, A: np.ndarray, a_lbl: str, B: np.ndarray, b_lbl: str,
             alpha: float, beta: float, cmask: Optional[np.ndarray] = None) -> np.ndarray:
    """Same sums as contract_naive (bit-identical; pinned by a test), with the operands first
    copied into [free][contracted] order so the inner loop is contiguous (memory order only)."""
    L = analyse_labels(c_lbl, a_lbl, b_lbl)
    fa = [x for x in c_lbl if x in a_lbl]
    fb = [x for x in c_lbl if x in b_lbl]
    A2 = np.ascontiguousarray(np.transpose(A, [a_lbl.index(x) for x in fa + L.con]))
    B2 = np.ascontiguousarray(np.transpose(B, [b_lbl.index(x) for x in fb + L.con]))
    nfa = int(np.prod([A.shape[a_lbl.index(x)] for x in fa], dtype=np.int64))
    nfb = int(np.prod([B.shape[b_lbl.index(x)] for x in fb], dtype=np.int64))
    K = int(np.prod([A.shape[a_lbl.index(x)] for x in L.con], dtype=np.int64))
    P = np.empty(nfa * nfb, dtype=np.float64)
    A2f, B2f = _lib.f64(A2.reshape(-1)), _lib.f64(B2.reshape(-1))
    _lib.lib().orc_contract_gathered(nfa, nfb, K, _lib.ptr(A2f, ctypes.c_double),
                                     _lib.ptr(B2f, ctypes.c_double), _lib.ptr(P, ctypes.c_double))
    shp_fa = [A.shape[a_lbl.index(x)] for x in fa]
    shp_fb = [B.shape[b_lbl.index(x)] for x in fb]
    Pt = P.reshape(shp_fa + shp_fb)
    S = np.transpose(Pt, [(fa + fb).index(x) for x in c_lbl])   # memory order only
    AS = alpha * S
    out = np.array(C, dtype=np.float64, copy=True)
    if beta == 0.0:
        new = np.array(AS)  # "=" : C is not read (reading R3)
    else:
        new = beta * out + AS
    if cmask is None:
        return np.ascontiguousarray(new)
    return np.ascontiguousarray(np.where(cmask.astype(bool), new, out))


def contract3_naive(C: np.ndarray, c_lbl: str, A: np.ndarray, a_lbl: str, B: np.ndarray, b_lbl: str,
                    D: np.ndarray, d_lbl: str, alpha: float, beta: float,
                    cmask: Optional[np.ndarray] = None) -> np.ndarray:
    """PAPER Eq. cc9 evaluated as written (P293-300): C <- beta*C + alpha*sum A*B*D over every label not
    in C, one product per combination of label values -- the unfactorized loop (oracle.c
    orc_contract3_naive).  Each label must appear in exactly two of C, A, B, D.  Returns a new C."""
    lbls = (c_lbl, a_lbl, b_lbl, d_lbl)
    for l in lbls:
        for x in l:
            if sum(x in q for q in lbls) != 2:
                raise ValueError(f"label {x} must appear in exactly two operands")
    ext = {}
    for arr, lbl in ((C, c_lbl), (A, a_lbl), (B, b_lbl), (D, d_lbl)):
        for n, x in zip(arr.shape, lbl):
            if ext.setdefault(x, n) != n:
                raise ValueError(f"extent mismatch on label {x}")
    summed = []
    for l in (a_lbl, b_lbl, d_lbl):
        for x in l:
            if x not in c_lbl and x not in summed:
                summed.append(x)
    st = [_strides(X.shape) for X in (C, A, B, D)]

    def strides_of(labels, k):
        return _lib.i64([st[k][lbls[k].index(x)] if x in lbls[k] else 0 for x in labels] or [0])

    ext_f = _lib.i64([ext[x] for x in c_lbl])
    ext_k = _lib.i64([ext[x] for x in summed] or [1])
    sf = [strides_of(c_lbl, k) for k in range(4)]
    sk = [strides_of(summed, k) for k in range(1, 4)]
    Co = _lib.f64(C).copy()
    Ao, Bo, Do = _lib.f64(A), _lib.f64(B), _lib.f64(D)
    m = None if cmask is None else np.ascontiguousarray(cmask, dtype=np.uint8)
    P64, PD = ctypes.c_int64, ctypes.c_double
    _lib.lib().orc_contract3_naive(len(c_lbl), _lib.ptr(ext_f, P64), *[_lib.ptr(x, P64) for x in sf], len(summed),
                                   _lib.ptr(ext_k, P64), *[_lib.ptr(x, P64) for x in sk], _lib.ptr(Co, PD),
                                   _lib.ptr(Ao, PD), _lib.ptr(Bo, PD), _lib.ptr(Do, PD),
                                   None if m is None else _lib.ptr(m, ctypes.c_uint8), float(alpha), float(beta))
    return Co


def slice_of(D: np.ndarray, ranges) -> np.ndarray:
    """P159 "operations on different slices of the underlying allocated tensor": the sub-array over the
    index ranges [(begin, end)] of each dimension (a numpy view: writes go to D)."""
    return D[tuple(slice(b, e) for b, e in ranges)]


def add(C: np.ndarray, c_lbl: str, A: np.ndarray, a_lbl: str, alpha: float, beta: float,
        cmask: Optional[np.ndarray] = None) -> np.ndarray:
    """P173 ``A(i,l) += alpha * D(l,i)``: C[x] <- beta*C[x] + alpha*A[pi(x)] (beta=0: C not read)."""
    if sorted(c_lbl) != sorted(a_lbl) or len(set(c_lbl)) != len(c_lbl):
        raise ValueError("add needs a label permutation")
    Ap = np.transpose(A, [a_lbl.index(x) for x in c_lbl])
    new = alpha * Ap if beta == 0.0 else beta * C + alpha * Ap
    if cmask is None:
        return np.ascontiguousarray(new, dtype=np.float64)
    return np.ascontiguousarray(np.where(cmask.astype(bool), new, C), dtype=np.float64)


def set_(C: np.ndarray, alpha: float, cmask: Optional[np.ndarray] = None) -> np.ndarray:
    """P172 ``A(i,l) = alpha``."""
    if cmask is None:
        return np.full(C.shape, float(alpha))
    return np.where(cmask.astype(bool), float(alpha), C)


def scalar(A: np.ndarray, a_lbl: str, B: np.ndarray, b_lbl: str, alpha: float) -> float:
    """Order-0 contraction s = alpha * sum_x A[x]*B[pi(x)], sequential over A's row-major order."""
    if sorted(a_lbl) != sorted(b_lbl):
        raise ValueError("scalar contraction needs matching label sets")
    Bp = np.ascontiguousarray(np.transpose(B, [b_lbl.index(x) for x in a_lbl]), dtype=np.float64)
    Af = _lib.f64(A.reshape(-1))
    Bf = Bp.reshape(-1)
    s = _lib.lib().orc_dot(Af.size, _lib.ptr(Af, ctypes.c_double), _lib.ptr(Bf, ctypes.c_double))
    return float(alpha) * s


def dots(a_rows: np.ndarray, b_rows: np.ndarray) -> np.ndarray:
    """Independent sequential dot products of matching rows (sampled output elements)."""
    a, b = _lib.f64(a_rows), _lib.f64(b_rows)
    n, K = a.shape
    out = np.empty(n, dtype=np.float64)
    _lib.lib().orc_dots(n, K, _lib.ptr(a, ctypes.c_double), _lib.ptr(b, ctypes.c_double),
                        _lib.ptr(out, ctypes.c_double))
    return out


def matvec(M: np.ndarray, x: np.ndarray) -> np.ndarray:
    Mf, xf = _lib.f64(M), _lib.f64(x)
    y = np.empty(Mf.shape[0], dtype=np.float64)
    _lib.lib().orc_matvec(Mf.shape[0], Mf.shape[1], _lib.ptr(Mf, ctypes.c_double),
                          _lib.ptr(xf, ctypes.c_double), _lib.ptr(y, ctypes.c_double))
    return y


# ----------------------------------------------------------------------------- sampled elements

def sampled_elements(c_idx: np.ndarray, c_lbl: str, a_lbl: str, b_lbl: str, ext: dict,
                     a_values, b_values, a_nz_elem=None, b_nz_elem=None) -> np.ndarray:
    """sum_y A[x_A, y] * B[x_B, y] for each global C index tuple in ``c_idx`` ([n, order]).

    ``a_values(idx)`` / ``b_values(idx)`` return the operand values at global index tuples
    (e.g. the seeded generator of ``synthetic``); ``*_nz_elem(idx)`` return 0/1 for zero-block
    masking (S216).  Contracted tuples in order of first appearance in A, row-major (R12)."""
    L = analyse_labels(c_lbl, a_lbl, b_lbl)
    kext = [ext[x] for x in L.con]
    grids = np.meshgrid(*[np.arange(n) for n in kext], indexing="ij")
    kidx = {x: g.reshape(-1) for x, g in zip(L.con, grids)}
    K = int(np.prod(kext, dtype=np.int64)) if kext else 1
    out = np.empty(len(c_idx), dtype=np.float64)
    for r, x in enumerate(np.asarray(c_idx)):
        lab = {l: np.full(K, int(v), dtype=np.int64) for l, v in zip(c_lbl, x)}
        lab.update(kidx)
        ia = np.stack([lab[l] for l in a_lbl], axis=-1)
        ib = np.stack([lab[l] for l in b_lbl], axis=-1)
        av, bv = a_values(ia), b_values(ib)
        if a_nz_elem is not None:
            av = np.where(a_nz_elem(ia) != 0, av, 0.0)
        if b_nz_elem is not None:
            bv = np.where(b_nz_elem(ib) != 0, bv, 0.0)
        out[r] = dots(av[None, :], bv[None, :])[0]
    return out


def cholesky_v(X: np.ndarray) -> np.ndarray:
    """PAPER Eq. cc12 (P312-318) as printed (reading R19):
        v(p,q,r,s) = sum_L X(p,r,L) X(q,s,L) - X(p,s,L) X(q,r,L)
    Two oracle contractions over L (sequential sums)."""
    n = X.shape[0]
    V = contract(np.zeros((n, n, n, n)), "pqrs", X, "prL", X, "qsL", 1.0, 0.0)
    return contract(V, "pqrs", X, "psL", X, "qrL", -1.0, 1.0)


def cholesky_v_row(Xa: np.ndarray, Xb: np.ndarray) -> np.ndarray:
    """PAPER Eq. cc12 at one fixed (p,q) = (a,b) (reading R19), for sampled checks at sizes where V
    cannot be formed:  v(a,b,r,s) = sum_L X(a,r,L) X(b,s,L) - X(a,s,L) X(b,r,L)
    with Xa = X(a,:,:), Xb = X(b,:,:) dense [n, N_L].  Two matrix products over L."""
    return Xa @ Xb.T - Xb @ Xa.T


def ladder_sample(vrow: np.ndarray, Tij: np.ndarray, alpha: float) -> float:
    """One output element of the ladder R(a,b,i,j) = alpha * sum_{r,s} v(a,b,r,s) T(r,s,i,j) (beta = 0),
    vrow = v(a,b,:,:), Tij = T(:,:,i,j); sequential-order sum over r then s."""
    return alpha * float(np.sum(vrow * Tij))



# ----------------------------------------------------------------------------- Freivalds check

def freivalds(c_blk: np.ndarray, c_lbl: str, a_sub: np.ndarray, a_lbl: str, b_sub: np.ndarray, b_lbl: str,
              x: np.ndarray, alpha: float, beta: float, c0_blk: np.ndarray):
    """SURVEY §8(c) step 5 (Freivalds): for one output block C_blk = beta*C0 + alpha*sum A.B, with
    x random over the C labels that come from B, returns (C_blk . x, beta*C0 . x + alpha*A.(B.x)).
    a_sub / b_sub are the operands restricted to the block's free index ranges (all contracted
    indices, zero blocks zero).  O(|A| + |B|) instead of O(|C| K); a wrong element of C changes the
    left side for almost every x.  Products by numpy.einsum (a library primitive)."""
    nb = "".join(l for l in c_lbl if l in b_lbl)
    na = "".join(l for l in c_lbl if l in a_lbl)
    con = "".join(l for l in a_lbl if l in b_lbl)
    y = np.einsum(f"{b_lbl},{nb}->{con}", b_sub, x)
    z = np.einsum(f"{a_lbl},{con}->{na}", a_sub, y)
    lhs = np.einsum(f"{c_lbl},{nb}->{na}", c_blk, x)
    rhs = beta * np.einsum(f"{c_lbl},{nb}->{na}", c0_blk, x) + alpha * z
    return lhs, rhs
