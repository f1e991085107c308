"""Sampled CCSD residual elements at full size -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

At BASELINE configs[3] size (O=100, V=800, N_L=1800) the literal transcription oracle/ccsd.py cannot
run (it forms every <pq||rs>, 3.3e11 elements for V_vvvv alone).  This module evaluates single
elements R1(a,i) and R2(a,b,i,j) of the SAME equations (Stanton-Gauss, oracle/ccsd.py's term list and
order of terms) directly from the seeded input recipe (reading R30), regenerating only the input
slices an element needs (synthetic/ counter generator by global index, spin maps of reading R7) and
evaluating each integral slice by Eq. cc12, <pq||rs> = sum_L X(p,r,L) X(q,s,L) - X(p,s,L) X(q,r,L),
with the sum over L taken after the other contraction it meets (a change of summation order only;
numpy/BLAS matrix products are the library primitives).  It shares nothing with the product.

Pinned in tests/test_ccsd_iteration.py: on mini shapes every element equals oracle.ccsd.iterate
(itself pinned to the second-quantized projections) within 1e-12.

Cost per element group: O(V^2 O N_L) for the F and W slices (about 1e11-1e12 FLOPs at configs[3]).
"""
from __future__ import annotations

import numpy as np

import synthetic as S


class Inputs:
    """The iteration's inputs (R30 recipe over the seeded raw blocks, spin maps of R6/R7) by slice."""

    TAGS = {"foo": 11, "fvv": 12, "fov": 19, "T1": 13, "T2": 14, "Xoo": 20, "Xov": 21, "Xvv": 18}

    def __init__(self, nO: int, nV: int, NL: int, seed: int):
        self.nO, self.nV, self.NL, self.seed = nO, nV, NL, seed
        self.so = np.where(np.arange(nO) < nO // 2, 1, -1)
        self.sv = np.where(np.arange(nV) < nV // 2, 1, -1)

    def _grid(self, name, shape, axes):
        """raw generator values of tensor ``name`` (dense shape ``shape``) on the grid of index arrays."""
        axes = [np.arange(n) if a is None else np.atleast_1d(np.asarray(a, dtype=np.int64)) for a, n in zip(axes, shape)]
        g = np.zeros([len(a) for a in axes], dtype=np.int64)
        for d, a in enumerate(axes):
            sh = [1] * len(axes)
            sh[d] = len(a)
            g = g * int(shape[d]) + a.reshape(sh)
        return S.values(self.seed, self.TAGS[name], g), axes

    def _spin(self, kinds, axes):
        s = [(self.so if k == "o" else self.sv)[a] for k, a in zip(kinds, axes)]
        sh = lambda d: [len(axes[x]) if x == d else 1 for x in range(len(axes))]   # noqa: E731
        return [s[d].reshape(sh(d)) for d in range(len(axes))]

    def T2(self, a=None, b=None, i=None, j=None):
        nO, nV = self.nO, self.nV
        v, ax = self._grid("T2", (nV, nV, nO, nO), (a, b, i, j))
        sa, sb, si, sj = self._spin("vvoo", ax)
        return np.where(sa + sb == si + sj, v, 0.0)

    def _pair(self, name, kinds, shape, axes):
        v, ax = self._grid(name, shape, axes)
        s0, s1 = self._spin(kinds, ax[:2])[:2]
        m = (s0 == s1)
        if len(shape) == 3:
            m = m[..., None]
        return np.where(m, v, 0.0)

    def T1(self):
        return self._pair("T1", "vo", (self.nV, self.nO), (None, None))

    def fov(self):
        return self._pair("fov", "ov", (self.nO, self.nV), (None, None))

    def foo(self):
        r = self._pair("foo", "oo", (self.nO, self.nO), (None, None))
        return 0.5 * (r + r.T)

    def fvv(self):
        r = self._pair("fvv", "vv", (self.nV, self.nV), (None, None))
        return 0.5 * (r + r.T)

    def Xoo(self):
        r = self._pair("Xoo", "oo", (self.nO, self.nO, self.NL), (None, None, None))
        return 0.5 * (r + r.transpose(1, 0, 2))

    def Xov(self):
        return self._pair("Xov", "ov", (self.nO, self.nV, self.NL), (None, None, None))

    def Xvv_rows(self, rows):
        """X_vv(a,:,:) for a in rows: (R(a,e,L) + R(e,a,L)) / 2."""
        nV, NL = self.nV, self.NL
        r1 = self._pair("Xvv", "vv", (nV, nV, NL), (rows, None, None))
        r2 = self._pair("Xvv", "vv", (nV, nV, NL), (None, rows, None)).transpose(1, 0, 2)
        return 0.5 * (r1 + r2)


class Sampler:
    """Element evaluator; caches the O(o v N_L) globals and the per-index slices it builds."""

    def __init__(self, inp: Inputs):
        self.inp = inp
        self.T1 = inp.T1()
        self.fov = inp.fov()
        self.foo = inp.foo()
        self.fvv = inp.fvv()
        self.Xoo = inp.Xoo()
        self.Xov = inp.Xov()                                   # (m, e, L); X_vo(b,j,L) = X_ov(j,b,L)
        # g(L) = sum_mf t_m^f X(m,f,L); Y2(m,j,L) = sum_f X(m,f,L) t_j^f
        self.g = np.einsum("fm,mfL->L", self.T1, self.Xov, optimize=True)
        self.Y2 = np.einsum("mfL,fj->mjL", self.Xov, self.T1, optimize=True)
        # F_me = f_me + sum_nf t_n^f <mn||ef>,  <mn||ef> = X(m,e)X(n,f) - X(m,f)X(n,e)
        self.Fme = (self.fov + np.einsum("meL,L->me", self.Xov, self.g, optimize=True)
                    - np.einsum("mnL,neL->me", self.Y2, self.Xov, optimize=True))
        self._xv, self._fae, self._fmi, self._wo, self._wab, self._wr = {}, {}, {}, {}, {}, {}
        self._t2 = {}
        nO, nV, NL = inp.nO, inp.nV, inp.NL
        # two more layouts of X_ov so that every large contraction is one matrix product (BLAS):
        # XT[e, m, L] = X_ov(m, e, L) and XL[L, m, e]
        self.XT = np.ascontiguousarray(self.Xov.transpose(1, 0, 2))
        self.XL = np.ascontiguousarray(self.Xov.transpose(2, 0, 1))
        self.XTm = self.XT.reshape(nV * nO, NL)                  # rows (e, m)
        self.XTv = self.XT.reshape(nV, nO * NL)                  # X_ov(m, e, L) as [e][(m, L)]

    def t2_i(self, i):
        """t_in^ef as (e, f, n) for one i (cached: the largest slice, V^2 O)."""
        if i not in self._t2:
            self._t2[i] = self.inp.T2(i=[i])[:, :, 0, :]
        return self._t2[i]

    def _xe(self, C):
        """sum_{m,L} X_ov(m, e, L) C(m, L) for all e."""
        return self.XTv @ C.reshape(-1)

    # ---------------------------------------------------------------------------------- slices
    def xv(self, a):
        if a not in self._xv:
            self._xv[a] = self.inp.Xvv_rows([a])[0]            # X_vv(a, :, L)
        return self._xv[a]

    def yt(self, b):
        """sum_m t_m^b X_ov(m, :, L)."""
        nO, nV, NL = self.inp.nO, self.inp.nV, self.inp.NL
        return (self.T1[b] @ self.Xov.reshape(nO, nV * NL)).reshape(nV, NL)

    def fae_row(self, a):
        """F_ae for one a (all e): f_ae - 1/2 f_me t_m^a + t_m^f <ma||fe> - 1/2 taut_mn^af <mn||ef>."""
        if a in self._fae:
            return self._fae[a]
        T1, Xov, Xa = self.T1, self.Xov, self.xv(a)
        r = self.fvv[a].copy()
        r -= 0.5 * self.fov.T @ T1[a]
        # <ma||fe> = X(m,f) X(a,e) - X(m,e) X(a,f)
        Ya = T1.T @ Xa                                         # (m, L): sum_f X(a,f,L) t_m^f
        r += Xa @ self.g - self._xe(Ya)
        # taut_mn^af = t_mn^af + 1/2 (t_m^a t_n^f - t_m^f t_n^a), index order (f, m, n)
        tt = self.inp.T2(a=[a])[0] + 0.5 * (np.einsum("m,fn->fmn", T1[a], T1, optimize=True) - np.einsum("fm,n->fmn", T1, T1[a], optimize=True))
        nO, nV = self.inp.nO, self.inp.nV
        C1 = tt.transpose(1, 0, 2).reshape(nO, nV * nO) @ self.XTm   # sum_fn t(f,m,n) X(n,f,L)
        C2 = tt.transpose(2, 0, 1).reshape(nO, nV * nO) @ self.XTm   # sum_fm t(f,m,n) X(m,f,L)
        r -= 0.5 * (self._xe(C1) - self._xe(C2))
        self._fae[a] = r
        return r

    def fmi_col(self, i):
        """F_mi for one i (all m): f_mi + 1/2 t_i^e f_me + t_n^e <mn||ie> + 1/2 taut_in^ef <mn||ef>."""
        if i in self._fmi:
            return self._fmi[i]
        T1, Xov, Xoo = self.T1, self.Xov, self.Xoo
        r = self.foo[:, i].copy()
        r += 0.5 * self.fov @ T1[:, i]
        # <mn||ie> = X(m,i) X(n,e) - X(m,e) X(n,i)
        nV, nO, NL = self.inp.nV, self.inp.nO, self.inp.NL
        Xmv = Xov.reshape(nO, nV * NL)                              # X_ov as [m][(e, L)]
        v = T1 @ Xoo[:, i, :]                                       # (e, L): sum_n t_n^e X(n,i,L)
        r += Xoo[:, i, :] @ self.g - Xmv @ v.reshape(-1)
        # taut_in^ef (e, f, n)
        tt = self.t2_i(i) + 0.5 * (np.einsum("e,fn->efn", T1[:, i], T1, optimize=True) - np.einsum("f,en->efn", T1[:, i], T1, optimize=True))
        A = tt.reshape(nV, nV * nO) @ self.XTm                      # sum_fn t(e,f,n) X(n,f,L)
        B = tt.transpose(1, 0, 2).reshape(nV, nV * nO) @ self.XTm   # sum_en t(e,f,n) X(n,e,L)
        r += 0.5 * (Xmv @ A.reshape(-1) - Xmv @ B.reshape(-1))
        self._fmi[i] = r
        return r

    def tau(self, a=None, b=None, i=None, j=None):
        T1 = self.T1
        t = self.inp.T2(a, b, i, j)
        ax = lambda x, n: np.arange(n) if x is None else np.atleast_1d(x)   # noqa: E731
        A, B_, I, J = ax(a, self.inp.nV), ax(b, self.inp.nV), ax(i, self.inp.nO), ax(j, self.inp.nO)
        t = t + np.einsum("ai,bj->abij", T1[np.ix_(A, I)], T1[np.ix_(B_, J)], optimize=True) \
              - np.einsum("bi,aj->abij", T1[np.ix_(B_, I)], T1[np.ix_(A, J)], optimize=True)
        return t

    def wmnij(self, i, j):
        """W_mnij for one (i,j): <mn||ij> + P(ij) t_j^e <mn||ie> + 1/4 tau_ij^ef <mn||ef>."""
        if (i, j) in self._wo:
            return self._wo[(i, j)]
        Xoo, Xov, Y2 = self.Xoo, self.Xov, self.Y2
        w = Xoo[:, i, :] @ Xoo[:, j, :].T - Xoo[:, j, :] @ Xoo[:, i, :].T
        # t_j^e <mn||ie> = X(m,i) Y2(n,j) - Y2(m,j) X(n,i) ; minus the same with i <-> j
        w += Xoo[:, i, :] @ Y2[:, j, :].T - Y2[:, j, :] @ Xoo[:, i, :].T
        w -= Xoo[:, j, :] @ Y2[:, i, :].T - Y2[:, i, :] @ Xoo[:, j, :].T
        tij = self.tau(i=i, j=j)[:, :, 0, 0]
        Am = np.einsum("Lmf,Lnf->mn", np.matmul(self.XL, tij), self.XL, optimize=True)   # sum X(m,e) t(e,f) X(n,f)
        w += 0.25 * (Am - Am.T)
        self._wo[(i, j)] = w
        return w

    def wabef(self, a, b):
        """W_abef for one (a,b): <ab||ef> - P(ab) t_m^b <am||ef> + 1/4 tau_mn^ab <mn||ef>."""
        if (a, b) in self._wab:
            return self._wab[(a, b)]
        Xa, Xb, Xov = self.xv(a), self.xv(b), self.Xov
        P = Xa @ Xb.T
        w = P - P.T
        Q1 = Xa @ self.yt(b).T            # sum_m t_m^b X(a,e) X(m,f)
        Q2 = Xb @ self.yt(a).T
        w -= Q1 - Q1.T
        w += Q2 - Q2.T
        tab = self.tau(a=a, b=b)[0, 0]
        nO, nV, NL = self.inp.nO, self.inp.nV, self.inp.NL
        Z = (tab.T @ Xov.reshape(nO, nV * NL)).reshape(nO, nV, NL)           # sum_m t(m,n) X(m,e,L)
        Bm = np.ascontiguousarray(Z.transpose(1, 0, 2)).reshape(nV, nO * NL) @ self.XTv.T
        w += 0.25 * (Bm - Bm.T)
        self._wab[(a, b)] = w
        return w

    def wmbej(self, b, j):
        """W_mbej for one (b,j) (all m, e): <mb||ej> + t_j^f <mb||ef> - t_n^b <mn||ej>
        - (1/2 t_jn^fb + t_j^f t_n^b) <mn||ef>."""
        if (b, j) in self._wr:
            return self._wr[(b, j)]
        T1, Xov, Xoo, Y2, Xb = self.T1, self.Xov, self.Xoo, self.Y2, self.xv(b)
        xvo = Xov[j, b, :]                                   # X_vo(b,j,L)
        w = Xov @ xvo - Xoo[:, j, :] @ Xb.T                  # <mb||ej> = X(m,e) X(b,j) - X(m,j) X(b,e)
        ybj = Xb.T @ T1[:, j]                                # sum_f X(b,f,L) t_j^f
        w += Xov @ ybj - Y2[:, j, :] @ Xb.T                  # <mb||ef> = X(m,e) X(b,f) - X(m,f) X(b,e)
        u = T1[b] @ Xoo[:, j, :]                             # sum_n t_n^b X(n,j,L)
        w -= Xov @ u - Xoo[:, j, :] @ self.yt(b).T           # <mn||ej> = X(m,e) X(n,j) - X(m,j) X(n,e)
        tq = 0.5 * self.inp.T2(b=[b], i=[j])[:, 0, 0, :] + np.outer(T1[:, j], T1[b])   # t_jn^fb at (f, n)
        wv = self.XTm.T @ tq.reshape(-1)                                # sum_nf t(f,n) X(n,f,L)
        U = np.matmul(self.XL, tq)                                      # (L, m, n): sum_f X(m,f,L) t(f,n)
        w -= Xov @ wv - np.einsum("Lmn,Lne->me", U, self.XL, optimize=True)
        self._wr[(b, j)] = w
        return w

    # ---------------------------------------------------------------------------------- residuals
    def r1(self, a, i):
        T1, Xov, Xoo = self.T1, self.Xov, self.Xoo
        Xa = self.xv(a)
        r = self.fov[i, a]
        r += T1[:, i] @ self.fae_row(a)
        r -= T1[a] @ self.fmi_col(i)
        t_a_i = self.inp.T2(a=[a], i=[i])[0, :, 0, :]        # (e, m)
        r += np.einsum("em,me->", t_a_i, self.Fme, optimize=True)
        # - t_n^f <na||if>,  <na||if> = X(n,i) X(a,f) - X(n,f) X(a,i)
        Ya = np.einsum("fL,fn->nL", Xa, T1, optimize=True)
        r -= np.einsum("nL,nL->", Xoo[:, i, :], Ya, optimize=True) - self.g @ Xov[i, a, :]
        # - 1/2 t_im^ef <ma||ef>,  <ma||ef> = X(m,e) X(a,f) - X(m,f) X(a,e)
        ti = self.t2_i(i)                                     # (e, f, m)
        nO, nV = self.inp.nO, self.inp.nV
        Q = ti.transpose(1, 0, 2).reshape(nV, nV * nO) @ self.XTm    # sum_em t(e,f,m) X(m,e,L)
        Qp = ti.reshape(nV, nV * nO) @ self.XTm                      # sum_fm t(e,f,m) X(m,f,L)
        r -= 0.5 * (np.einsum("fL,fL->", Xa, Q, optimize=True) - np.einsum("eL,eL->", Xa, Qp, optimize=True))
        # - 1/2 t_mn^ae <nm||ei>,  <nm||ei> = X(n,e) X(m,i) - X(n,i) X(m,e)
        ta = self.inp.T2(a=[a])[0]                            # (e, m, n)
        K1 = ta.transpose(1, 0, 2).reshape(nO, nV * nO) @ self.XTm   # sum_en t(e,m,n) X(n,e,L)
        K2 = ta.transpose(2, 0, 1).reshape(nO, nV * nO) @ self.XTm   # sum_em t(e,m,n) X(m,e,L)
        r -= 0.5 * (np.einsum("mL,mL->", K1, Xoo[:, i, :], optimize=True) - np.einsum("nL,nL->", K2, Xoo[:, i, :], optimize=True))
        return float(r)

    def _zab(self, a, b, i, j):
        """t_ij^ae (F_be - 1/2 t_m^b F_me) - t_m^a <mb||ij>."""
        T1, Xoo, Xov = self.T1, self.Xoo, self.Xov
        fbe = self.fae_row(b) - 0.5 * T1[b] @ self.Fme
        z = self.inp.T2(a=[a], i=[i], j=[j])[0, :, 0, 0] @ fbe
        mb = Xoo[:, i, :] @ Xov[j, b, :] - Xoo[:, j, :] @ Xov[i, b, :]     # <mb||ij> over m
        return z - T1[a] @ mb

    def _zij(self, a, b, i, j):
        """- t_im^ab (F_mj + 1/2 t_j^e F_me) + t_i^e <ab||ej>."""
        T1, Xov = self.T1, self.Xov
        fmj = self.fmi_col(j) + 0.5 * self.Fme @ T1[:, j]
        z = -(self.inp.T2(a=[a], b=[b], i=[i])[0, 0, 0, :] @ fmj)
        ab = self.xv(a) @ Xov[j, b, :] - self.xv(b) @ Xov[j, a, :]        # <ab||ej> over e
        return z + T1[:, i] @ ab

    def _zr(self, a, b, i, j):
        """t_im^ae W_mbej - t_i^e t_m^a <mb||ej>."""
        T1, Xov, Xoo = self.T1, self.Xov, self.Xoo
        z = np.einsum("em,me->", self.inp.T2(a=[a], i=[i])[0, :, 0, :], self.wmbej(b, j), optimize=True)
        mbej = Xov @ Xov[j, b, :] - Xoo[:, j, :] @ self.xv(b).T           # <mb||ej> (m, e)
        return z - T1[a] @ mbej @ T1[:, i]

    def r2(self, a, b, i, j):
        Xov = self.Xov
        r = Xov[i, a, :] @ Xov[j, b, :] - Xov[i, b, :] @ Xov[j, a, :]      # <ij||ab>
        r += self._zab(a, b, i, j) - self._zab(b, a, i, j)
        r += self._zij(a, b, i, j) - self._zij(a, b, j, i)
        r += 0.5 * np.sum(self.tau(a=a, b=b)[0, 0] * self.wmnij(i, j))
        r += 0.5 * np.sum(self.tau(i=i, j=j)[:, :, 0, 0] * self.wabef(a, b))
        r += self._zr(a, b, i, j) - self._zr(b, a, i, j) - self._zr(a, b, j, i) + self._zr(b, a, j, i)
        return float(r)

    def nonzero_r2(self, a, b, i, j):
        s = self.inp
        return s.sv[a] + s.sv[b] == s.so[i] + s.so[j]

    def nonzero_r1(self, a, i):
        return self.inp.sv[a] == self.inp.so[i]
