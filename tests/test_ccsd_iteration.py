"""Synthetic CCSD iteration (configs[3] structure, reading R18): the product driver (Scheduler over libtt,
>= 3-virtual integrals factorized through the Cholesky vectors, the ladder through the implicit operand)
vs the oracle's literal Stanton-Gauss transcription with explicit integrals (oracle/ccsd.py), on small
spin-sparse shapes with ragged tiles, several batches of the implicit ladder and split-K terms.

The oracle side builds its tensors from its own copy of the maps below (classes, spin rules, input tags
of the synthetic recipe), not from the product's TENSORS."""
import numpy as np
import pytest

import synthetic as S
from oracle import layout as L
from oracle import ops as O

# oracle-side spec: name -> (index classes, spin split, input tag); outputs have tag None
SPEC = {
    "foo": ("oo", ([0], [1]), 11), "fvv": ("vv", ([0], [1]), 12), "fov": ("ov", ([0], [1]), 19),
    "T1": ("vo", ([0], [1]), 13), "T2": ("vvoo", ([0, 1], [2, 3]), 14),
    "Xoo": ("ooL", ([0], [1]), 20), "Xov": ("ovL", ([0], [1]), 21), "Xvv": ("vvL", ([0], [1]), 18),
    "R1": ("vo", ([0], [1]), None), "R2": ("vvoo", ([0, 1], [2, 3]), None),
}


def oracle_tensors(O_, V_, tO, tV, NL, tL):
    so = L.IndexSpace(O_, [(0, O_ // 2, 1), (O_ // 2, O_, -1)])
    sv = L.IndexSpace(V_, [(0, V_ // 2, 1), (V_ // 2, V_, -1)])
    tis = {"o": L.tile_fixed(so, tO), "v": L.tile_fixed(sv, tV), "L": L.tile_fixed(L.IndexSpace(NL), tL)}
    return {n: (L.tensor_spin([tis[c] for c in cls], up, lo), tag) for n, (cls, (up, lo), tag) in SPEC.items()}


def oracle_reference(shape, seed):
    from oracle import ccsd as OC
    ot = oracle_tensors(*shape)
    raw = {n: O.dense_masked(T, S.dense(T.shape, seed, tag)) for n, (T, tag) in ot.items() if tag is not None}
    masks = {n: O.nz_mask(T) for n, (T, tag) in ot.items() if tag is None}
    return ot, OC.iterate(OC.hermitian_inputs(raw), masks)


def _fock_ops(n):
    """Dense annihilation matrices a_p on the 2^n occupation basis (Jordan-Wigner signs: (-1)^(number
    of occupied orbitals below p))."""
    dim = 1 << n
    ops = []
    for p in range(n):
        a = np.zeros((dim, dim))
        for det in range(dim):
            if (det >> p) & 1:
                a[det ^ (1 << p), det] = -1.0 if bin(det & ((1 << p) - 1)).count("1") % 2 else 1.0
        ops.append(a)
    return ops


def test_oracle_ccsd_equals_second_quantized_projections():
    """The oracle's CCSD transcription against the DEFINITION: with H_N = sum_pq f_pq {a+_p a_q} +
    1/4 sum_pqrs <pq||rs> {a+_p a+_q a_s a_r} (normal order w.r.t. Phi, <pq||rs> from Eq. cc12) and
    T = sum t_i^a a+_a a_i + 1/4 sum t_ij^ab a+_a a+_b a_j a_i, the residuals are the projections
    R1(a,i) = <Phi_i^a| e^-T H_N e^T |Phi>, R2(a,b,i,j) = <Phi_ij^ab| e^-T H_N e^T |Phi>, and
    E = <Phi| e^-T H_N e^T |Phi>.  Evaluated with dense matrices on the 2^7 Fock space of 3 occupied +
    4 virtual spin-orbitals -- independent of the Stanton-Gauss expansion, so a wrong sign, factor or
    index in any term of oracle/ccsd.py fails here.  Inputs: the R30 recipe (symmetric X and f),
    antisymmetric T2 (T's operator sees only that part)."""
    from oracle import ccsd as OC
    nO, nV, NL = 3, 4, 5
    n = nO + nV
    rng = np.random.default_rng(11)
    raw = {"Xoo": rng.uniform(-1, 1, (nO, nO, NL)), "Xov": rng.uniform(-1, 1, (nO, nV, NL)),
           "Xvv": rng.uniform(-1, 1, (nV, nV, NL)), "foo": rng.uniform(-1, 1, (nO, nO)),
           "fvv": rng.uniform(-1, 1, (nV, nV)), "fov": rng.uniform(-1, 1, (nO, nV)),
           "T1": rng.uniform(-1, 1, (nV, nO))}
    t2 = rng.uniform(-1, 1, (nV, nV, nO, nO))
    t2 = t2 - t2.transpose(1, 0, 2, 3)
    raw["T2"] = t2 - t2.transpose(0, 1, 3, 2)
    D = OC.hermitian_inputs(raw)
    masks = {"R1": np.ones((nV, nO)), "R2": np.ones((nV, nV, nO, nO))}
    ref = OC.iterate(D, masks)
    V, o, v = OC.full_v(D)
    f = np.zeros((n, n))
    f[:nO, :nO], f[:nO, nO:], f[nO:, :nO], f[nO:, nO:] = D["foo"], D["fov"], D["fov"].T, D["fvv"]
    a = _fock_ops(n)
    c = [x.T for x in a]
    dim = 1 << n
    occ = np.zeros(dim)
    phi = (1 << nO) - 1
    occ[phi] = 1.0
    # H_N = sum f_pq {p+ q} + 1/4 sum v {p+ q+ s r}; by Wick's theorem the plain two-body operator is
    # 1/4 sum v {p+ q+ s r} + sum_pq (sum_i <pi||qi>) p+ q + const, so H_N = sum (f - gm) p+ q + V - const
    # with the constant fixed by <Phi|H_N|Phi> = 0
    gm = np.einsum("piqi->pq", V[:, :nO, :, :nO])
    H = np.zeros((dim, dim))
    for p in range(n):
        for q in range(n):
            H += (f[p, q] - gm[p, q]) * (c[p] @ a[q])
    for p in range(n):
        for q in range(n):
            for r in range(n):
                for s_ in range(n):
                    if V[p, q, r, s_] != 0.0:
                        H += 0.25 * V[p, q, r, s_] * (c[p] @ c[q] @ a[s_] @ a[r])
    H -= (occ @ H @ occ) * np.eye(dim)
    T = np.zeros((dim, dim))
    for i in range(nO):
        for A in range(nV):
            T += D["T1"][A, i] * (c[nO + A] @ a[i])
            for j in range(nO):
                for B in range(nV):
                    T += 0.25 * D["T2"][A, B, i, j] * (c[nO + A] @ c[nO + B] @ a[j] @ a[i])
    eT, emT, term = np.eye(dim), np.eye(dim), np.eye(dim)
    for k in range(1, 2 * nO + 1):      # T is nilpotent
        term = term @ T / k
        eT = eT + term
        emT = emT + (-1) ** k * term
    Hbar_phi = emT @ (H @ (eT @ occ))
    E = Hbar_phi[phi]
    assert abs(E - ref["E"]) <= 1e-12 * max(1.0, abs(E))
    for i in range(nO):
        for A in range(nV):
            ket = c[nO + A] @ a[i] @ occ
            assert abs(ket @ Hbar_phi - ref["R1"][A, i]) <= 1e-11, ("R1", A, i)
    for i in range(nO):
        for j in range(nO):
            for A in range(nV):
                for B in range(nV):
                    ket = c[nO + A] @ c[nO + B] @ a[j] @ a[i] @ occ
                    assert abs(ket @ Hbar_phi - ref["R2"][A, B, i, j]) <= 1e-11, ("R2", A, B, i, j)


def test_oracle_ccsd_pins():
    """Pins of the oracle transcription (CPU): (1) T = 0 gives R1 = f_ov^T, R2 = <ij||ab>, E = 0 exactly;
    (2) the residuals are linear in the Fock matrix when the amplitudes are fixed (f enters linearly);
    (3) R2 is antisymmetric under a<->b and under i<->j (every term is antisymmetrized: <ij||ab> and the
    ladder by Eq. cc12's form, the rest by P(ab) / P(ij) or by tau's antisymmetry) when T2 is
    antisymmetric; (4) the energy equals its two textbook forms (1/4 <ij||ab> t2 + 1/2 <ij||ab> t1 t1
    when <ij||ab> is antisymmetric)."""
    from oracle import ccsd as OC
    shape = (6, 8, 3, 2, 10, 5)
    ot = oracle_tensors(*shape)
    D = OC.hermitian_inputs({n: O.dense_masked(T, S.dense(T.shape, 5, tag)) for n, (T, tag) in ot.items()
                             if tag is not None})
    masks = {n: O.nz_mask(T) for n, (T, tag) in ot.items() if tag is None}
    Vfull, o, v = OC.full_v(D)
    # (1) zero amplitudes
    D0 = dict(D, T1=np.zeros_like(D["T1"]), T2=np.zeros_like(D["T2"]))
    r0 = OC.iterate(D0, masks)
    assert np.array_equal(r0["R1"], np.where(masks["R1"].astype(bool), D["fov"].T, 0.0))
    assert np.array_equal(r0["R2"], np.where(masks["R2"].astype(bool), Vfull[o, o, v, v].transpose(2, 3, 0, 1), 0.0))
    assert r0["E"] == 0.0
    # (3) antisymmetric T2 -> antisymmetric R2
    T2 = D["T2"]
    T2a = T2 - T2.transpose(1, 0, 2, 3)
    T2a = T2a - T2a.transpose(0, 1, 3, 2)
    r = OC.iterate(dict(D, T2=T2a), masks)
    R2 = r["R2"]
    scale = np.abs(R2).max()
    assert np.abs(R2 + R2.transpose(1, 0, 2, 3)).max() <= 1e-12 * scale
    assert np.abs(R2 + R2.transpose(0, 1, 3, 2)).max() <= 1e-12 * scale
    # (2) f -> 2 f at fixed amplitudes: R(2f) - R(f) = R(f) - R(0 f)
    f0 = {k: np.zeros_like(D[k]) for k in ("foo", "fvv", "fov")}
    f2 = {k: 2 * D[k] for k in ("foo", "fvv", "fov")}
    rf, r2f, r0f = OC.iterate(D, masks), OC.iterate(dict(D, **f2), masks), OC.iterate(dict(D, **f0), masks)
    for k in ("R1", "R2"):
        s = np.abs(rf[k]).max()
        assert np.abs((r2f[k] - rf[k]) - (rf[k] - r0f[k])).max() <= 1e-12 * s
    # (4) energy forms with antisymmetric amplitudes
    T1 = D["T1"]
    oovv = Vfull[o, o, v, v]
    e_t2 = 0.25 * np.einsum("ijab,abij->", oovv, T2a)
    e_t1 = 0.5 * np.einsum("ijab,ai,bj->", oovv, T1, T1)
    e_f = np.einsum("ia,ai->", D["fov"], T1)
    assert abs(r["E"] - (e_f + e_t2 + e_t1)) <= 1e-12 * abs(r["E"])


def test_oracle_ccsd_ladder_factorization():
    """The product's factorization of 1/2 tau W_abef (T1-dressed Cholesky ladder + I_mnij terms, DESIGN
    §9) equals the oracle's explicit W_abef term, computed independently here with numpy.einsum
    (library routine) -- the algebra the driver relies on, checked on random inputs."""
    from oracle import ccsd as OC
    shape = (6, 8, 3, 2, 10, 5)
    ot = oracle_tensors(*shape)
    D = OC.hermitian_inputs({n: O.dense_masked(T, S.dense(T.shape, 7, tag)) for n, (T, tag) in ot.items()
                             if tag is not None})
    V, o, v = OC.full_v(D)
    T1, T2 = D["T1"], D["T2"]
    tau = T2 + np.einsum("ai,bj->abij", T1, T1) - np.einsum("bi,aj->abij", T1, T1)
    W = V[v, v, v, v] - np.einsum("bm,amef->abef", T1, V[v, o, v, v]) + np.einsum("am,bmef->abef", T1, V[v, o, v, v]) \
        + 0.25 * np.einsum("abmn,mnef->abef", tau, V[o, o, v, v])
    ref = 0.5 * np.einsum("efij,abef->abij", tau, W)
    Xh = D["Xvv"] - np.einsum("am,meL->aeL", T1, D["Xov"])
    Vh = np.einsum("aeL,bfL->abef", Xh, Xh) - np.einsum("afL,beL->abef", Xh, Xh)
    I = np.einsum("mnef,efij->mnij", V[o, o, v, v], tau)
    got = 0.5 * np.einsum("efij,abef->abij", tau, Vh) - 0.5 * np.einsum("am,bn,mnij->abij", T1, T1, I) \
        + 0.125 * np.einsum("abmn,mnij->abij", tau, I)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(8, 12, 2, 3, 10, 5), (12, 20, 3, 5, 14, 7), (14, 20, 3, 5, 14, 7),
                                   (10, 18, 3, 4, 22, 6)])
def test_ccsd_iteration_vs_oracle(shape):
    import torch
    import paper_2201_01257_b200 as tt
    from paper_2201_01257_b200.ccsd import CCSDIteration
    O_, V_, tO, tV, NL, tL = shape
    ctx = tt.Context(device=0, stream=torch.cuda.current_stream().cuda_stream)
    it = CCSDIteration(tt, ctx, O_, V_, tO, tV, NL, tL, seed=3, ws_gb=2e-5, nstreams=3)
    nlev, E = it.run()
    got = {n: it.T[n].download() for n in ("R1", "R2")}
    ctx.sync()
    ot, ref = oracle_reference(shape, 3)
    for n in ("R1", "R2"):
        r = O.pack(ot[n][0], ref[n])
        assert np.abs(got[n] - r).max() / np.abs(r).max() <= 1e-11, n
    assert abs(E - ref["E"]) <= 1e-11 * abs(ref["E"])
    assert nlev >= 10
    # a second run replays the cached plans and gives the same bits
    nlev2, E2 = it.run()
    got2 = {n: it.T[n].download() for n in ("R1", "R2")}
    ctx.sync()
    assert E2 == E and all(np.array_equal(got[n], got2[n]) for n in got)


@pytest.mark.parametrize("shape", [(6, 8, 3, 2, 10, 5), (8, 12, 2, 3, 10, 5)])
def test_sampled_elements_equal_literal_oracle(shape):
    """oracle/ccsd_sample.py (element-wise evaluation from the seeded recipe, integrals by Eq. cc12 with
    the L sum taken last -- the full-size checker) equals oracle.ccsd.iterate on every element."""
    from oracle.ccsd_sample import Inputs, Sampler
    O_, V_, tO, tV, NL, tL = shape
    ot, ref = oracle_reference(shape, 3)
    sm = Sampler(Inputs(O_, V_, NL, 3))
    s1 = np.abs(ref["R1"]).max()
    for a in range(V_):
        for i in range(O_):
            if sm.nonzero_r1(a, i):
                assert abs(sm.r1(a, i) - ref["R1"][a, i]) <= 1e-12 * s1, (a, i)
            else:
                assert ref["R1"][a, i] == 0.0
    s2 = np.abs(ref["R2"]).max()
    rng = np.random.default_rng(1)
    for _ in range(60):
        a, b = rng.integers(0, V_, 2)
        i, j = rng.integers(0, O_, 2)
        if sm.nonzero_r2(a, b, i, j):
            assert abs(sm.r2(a, b, i, j) - ref["R2"][a, b, i, j]) <= 1e-12 * s2, (a, b, i, j)
        else:
            assert ref["R2"][a, b, i, j] == 0.0
