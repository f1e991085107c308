"""Pins of the CPU oracle against things other than itself (paper values, closed forms, invariants,
an independent library routine).  CPU only.  Each test names what it pins and the passage."""
import json
import os
from itertools import product

import numpy as np
import pytest

import synthetic as S
from oracle import layout as L
from oracle import ops as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def rnd(shape, seed, tag=1, kind=S.KIND_UNIFORM):
    return S.dense(shape, seed, tag, kind)


def normwise(x, ref):
    return np.abs(x - ref).max() / max(np.abs(ref).max(), 1e-300)


# ------------------------------------------------------------------ generator

def test_splitmix64_reference_vectors():
    """synthetic.splitmix64 == the published splitmix64 seed-0 sequence (golden)."""
    g = np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        xs = np.array([0, g, g * np.uint64(2)], dtype=np.uint64)
    got = [format(int(v), "016x") for v in S.splitmix64(xs)]
    assert got == GOLD["splitmix64_seed0"]["outputs_hex"]


def test_generator_ranges():
    u = S.values(1, 4, np.arange(100000))
    assert u.min() >= -1.0 and u.max() < 1.0 and abs(u.mean()) < 0.02
    z = S.values(1, 4, np.arange(100000), S.KIND_INTEGER)
    assert set(np.unique(z)) == {-2.0, -1.0, 0.0, 1.0, 2.0}


# ------------------------------------------------------------------ tiling / layout (paper Fig. 2)

def fig2():
    f = GOLD["fig2"]
    N, M, K = L.IndexSpace(f["N"]), L.IndexSpace(f["M"]), L.IndexSpace(f["K"])
    return L.tile_fixed(N, f["tN_tile"]), L.tile_custom(M, f["tM_sizes"]), L.tile_fixed(K, f["tK_tile"])


def test_fig2_shapes():
    """P140: A{tM,tK} is 30x20 with eight blocks; tK four tiles of 5; tN ten tiles (P125)."""
    f = GOLD["fig2"]
    tN, tM, tK = fig2()
    assert tN.ntiles == f["tN_ntiles"] and tK.ntiles == f["tK_ntiles"]
    A = L.tensor_dense_map([tM, tK])
    assert list(A.shape) == f["A_shape"] and A.nblocks() == f["A_nblocks"]
    assert L.tensor_dense_map([tK, tN]).nblocks() == f["B_nblocks"]


def test_spec_block_extents():
    """S200-202."""
    g = GOLD["spec_block_extents"]
    tN, tM, tK = fig2()
    A = L.tensor_dense_map([tM, tK])
    assert list(A.block_extents(A.block_id([1, 0]))) == g["A_block_1_0"]
    assert list(A.block_extents(A.block_id([0, 3]))) == g["A_block_0_3"]
    assert list(L.tensor_dense_map([tN]).block_extents(9)) == g["tN_block_9"]


def test_tiling_rules():
    """S75-77 remainder rule, S85-87 coverage; spin ranges split tiles (S39)."""
    t = L.tile_fixed(L.IndexSpace(7), 3)
    assert [t.size(i) for i in range(t.ntiles)] == GOLD["spec_tiling"]["fixed_7_3"]
    assert L.tile_custom(L.IndexSpace(20), [20]).ntiles == 1
    with pytest.raises(L.OracleError):
        L.tile_custom(L.IndexSpace(20), [10, 5])
    sp = L.IndexSpace(150, [(0, 75, 1), (75, 150, -1)])
    t = L.tile_fixed(sp, 64)
    assert [t.size(i) for i in range(t.ntiles)] == [64, 11, 64, 11]
    assert t.tile_spin == [1, 1, -1, -1]
    with pytest.raises(L.OracleError):
        L.tile_custom(sp, [70, 80])  # straddles the spin boundary


def test_spin_example_2x2():
    """S191: one alpha and one beta tile per dim -> 2 of 4 blocks (spin conservation)."""
    sp = L.IndexSpace(4, [(0, 2, 1), (2, 4, -1)])
    t = L.tile_fixed(sp, 2)
    T = L.tensor_spin([t, t], [0], [1])
    assert sum(T.nz) == GOLD["spec_spin_2x2"]["nonzero_blocks"]
    assert T.nz == [1, 0, 0, 1]


def test_packed_layout_bijection():
    """Sparse-read law and addressing bijection (S216-217): pack/unpack round trip; 16-B starts;
    storage = sum of non-zero volumes (+ <=1 pad element per block)."""
    sp = L.IndexSpace(7, [(0, 3, 1), (3, 7, -1)])
    t = L.tile_fixed(sp, 2)      # tiles {2,1,2,2}
    T = L.tensor_spin([t, t, t], [0], [1, 2][:1])
    offs = T.blk_off()
    vols = [T.block_volume(b) for b in range(T.nblocks()) if T.nz[b]]
    assert all(o % 2 == 0 for o in offs if o >= 0)
    assert sum(vols) <= T.packed_elems() <= sum(vols) + len(vols) + 1
    P = np.arange(T.packed_elems(), dtype=np.float64) + 1.0
    D = O.unpack(T, P)
    P2 = O.pack(T, D)
    live = np.zeros_like(P, dtype=bool)
    for b, o in enumerate(offs):
        if o >= 0:
            live[o:o + T.block_volume(b)] = True
    assert np.array_equal(P2[live], P[live])
    # every stored element lands exactly once in the dense array, zero blocks stay zero
    assert np.count_nonzero(D) == live.sum()
    assert np.array_equal(np.sort(D[D != 0]), np.sort(P[live]))


def test_default_owner_round_robin():
    """P210 third scheme: round robin over non-zero blocks only."""
    sp = L.IndexSpace(4, [(0, 2, 1), (2, 4, -1)])
    t = L.tile_fixed(sp, 1)
    T = L.tensor_spin([t, t], [0], [1], nranks=3)
    own = T.owners()
    nzo = [o for o in own if o >= 0]
    assert nzo == [i % 3 for i in range(len(nzo))]
    assert all(o == -1 for o, z in zip(own, T.nz) if not z)


# ------------------------------------------------------------------ contraction values

CASES = [  # (c, a, b, extents)
    ("abij", "acik", "cbkj", dict(a=5, b=4, c=3, i=3, j=2, k=4)),      # ring (north_star)
    ("abij", "abcd", "cdij", dict(a=4, b=3, c=3, d=4, i=2, j=3)),      # ladder
    ("abij", "abkl", "klij", dict(a=3, b=4, k=3, l=2, i=3, j=2)),      # hole-hole
    ("ia", "il", "la", dict(i=6, l=5, a=7)),                           # Fig. 5 rule 7
    ("jbia", "kcai", "bjck", dict(a=3, b=4, c=2, i=3, j=2, k=3)),      # permuted labels
    ("ab", "acd", "dcb", dict(a=4, b=5, c=3, d=2)),
]


def _arrays(c, a, b, ext, seed, kind=S.KIND_UNIFORM):
    sh = lambda s: tuple(ext[x] for x in s)
    return rnd(sh(c), seed, 3, kind), rnd(sh(a), seed, 1, kind), rnd(sh(b), seed, 2, kind)


@pytest.mark.parametrize("case", CASES)
def test_contract_vs_einsum(case):
    """Independent library routine: numpy.einsum (no optimisation) on tiny shapes."""
    c, a, b, ext = case
    C, A, B = _arrays(c, a, b, ext, 7)
    ref = 1.0 * C + 0.75 * np.einsum(f"{a},{b}->{c}", A, B, optimize=False)
    got = O.contract(C, c, A, a, B, b, 0.75, 1.0)
    assert normwise(got, ref) < 1e-14


@pytest.mark.parametrize("case", CASES)
def test_naive_equals_gathered_bitwise(case):
    """The two oracle loop nests sum in the same order -> identical bits (reading R12)."""
    c, a, b, ext = case
    C, A, B = _arrays(c, a, b, ext, 3)
    r1 = O.contract_naive(C, c, A, a, B, b, -1.25, 0.5)
    r2 = O.contract(C, c, A, a, B, b, -1.25, 0.5)
    assert np.array_equal(r1, r2)


@pytest.mark.parametrize("case", CASES)
def test_integer_inputs_exact(case):
    """Integer-valued inputs: every partial sum is exact -> equals the int64 einsum exactly."""
    c, a, b, ext = case
    C, A, B = _arrays(c, a, b, ext, 5, S.KIND_INTEGER)
    ref = C.astype(np.int64) + 3 * np.einsum(f"{a},{b}->{c}", A.astype(np.int64), B.astype(np.int64))
    got = O.contract(C, c, A, a, B, b, 3.0, 1.0)
    assert np.array_equal(got, ref.astype(np.float64))


def test_linearity():
    c, a, b, ext = CASES[0]
    C, A, B = _arrays(c, a, b, ext, 11)
    A2 = rnd(A.shape, 12, 1)
    r = O.contract(C, c, A + A2, a, B, b, 1.0, 0.0)
    r1 = O.contract(C, c, A, a, B, b, 1.0, 0.0)
    r2 = O.contract(C, c, A2, a, B, b, 1.0, 0.0)
    assert normwise(r, r1 + r2) < 1e-14
    # alpha = 2 is an exact scaling; beta = 0 never reads C (NaN-safe, reading R3)
    Cn = np.full(C.shape, np.nan)
    assert np.array_equal(O.contract(Cn, c, A, a, B, b, 2.0, 0.0), 2.0 * r1)
    # alpha = 0 with beta = 1 leaves C unchanged (S491)
    assert np.array_equal(O.contract(C, c, A, a, B, b, 0.0, 1.0), C)


def test_label_permutation_equivalence():
    """Store A as A'(c,a,k,i) and relabel: same contraction -> identical bits."""
    c, a, b, ext = CASES[0]
    C, A, B = _arrays(c, a, b, ext, 13)
    Ap = np.ascontiguousarray(np.transpose(A, [1, 0, 3, 2]))  # acik -> caki
    r1 = O.contract(C, c, A, "acik", B, b, 1.5, -0.5)
    r2 = O.contract(C, c, Ap, "caki", B, b, 1.5, -0.5)
    assert np.array_equal(r1, r2)


def test_kronecker_identity():
    """B(c,b,k,j) = delta_cb delta_kj  =>  C = beta*C + alpha*A(a,b,i,j) exactly."""
    V, Oo = 6, 4
    A = rnd((V, V, Oo, Oo), 21)
    C = rnd((V, V, Oo, Oo), 21, 3)
    B = np.einsum("cb,kj->cbkj", np.eye(V), np.eye(Oo))
    got = O.contract(C, "abij", A, "acik", B, "cbkj", 0.5, 2.0)
    assert np.array_equal(got, 2.0 * C + 0.5 * A)


def test_rank1_closed_form():
    """A = x_a y_c z_i w_k, B = p_c q_b r_k s_j  =>  C = alpha*(y.p)(w.r) x_a q_b z_i s_j."""
    V, Oo = 7, 5
    x, y, p, q = (rnd((V,), s, 7) for s in (1, 2, 3, 4))
    z, w, r, s_ = (rnd((Oo,), s, 7) for s in (5, 6, 7, 8))
    A = np.einsum("a,c,i,k->acik", x, y, z, w)
    B = np.einsum("c,b,k,j->cbkj", p, q, r, s_)
    got = O.contract(np.zeros((V, V, Oo, Oo)), "abij", A, "acik", B, "cbkj", 1.25, 0.0)
    ref = 1.25 * float(y @ p) * float(w @ r) * np.einsum("a,b,i,j->abij", x, q, z, s_)
    assert normwise(got, ref) < 1e-14


def test_ladder_is_matmul():
    """Ladder = plain matmul after reshape (ab)x(cd) . (cd)x(ij)."""
    V, Oo = 5, 3
    Vt, T = rnd((V, V, V, V), 31, 4), rnd((V, V, Oo, Oo), 31, 5)
    got = O.contract(np.zeros((V, V, Oo, Oo)), "abij", Vt, "abcd", T, "cdij", 1.0, 0.0)
    ref = (Vt.reshape(V * V, V * V) @ T.reshape(V * V, Oo * Oo)).reshape(V, V, Oo, Oo)
    assert normwise(got, ref) < 1e-14


def test_spec_small_examples():
    """S490: 2x3 by 3x2 block = naive triple loop; S492 transpose add B[y][x] = A[x][y]."""
    A = np.array([[1., 2., 3.], [4., 5., 6.]])
    B = np.array([[7., 8.], [9., 10.], [11., 12.]])
    got = O.contract(np.zeros((2, 2)), "ij", A, "ik", B, "kj", 1.0, 0.0)
    assert np.array_equal(got, np.array([[58., 64.], [139., 154.]]))
    Bt = O.add(np.zeros((3, 2)), "li", A, "il", 1.0, 0.0)
    assert np.array_equal(Bt, A.T)


def test_fig5_program():
    """P194-198 (Fig. 5) with reading R2: A = 1, B = -1, C = 0.5*A.B -> -10.0 everywhere."""
    tN, tM, tK = fig2()
    A = O.set_(np.zeros((30, 20)), 1.0)                 # A(i,l) = 1.0   (rule 5)
    B = O.add(np.zeros((20, 100)), "la", -1.0 * np.ones((20, 100)), "la", 1.0, 1.0)  # B += -1.0*1
    C = O.contract(np.full((30, 100), np.nan), "ia", A, "il", B, "la", 0.5, 0.0)   # rule 7, "="
    assert np.all(C == GOLD["fig5"]["C_value"])


def test_scalar_contraction():
    """Order-0 result: rank-1 closed form, and the MP2-type energy sign (S641)."""
    x, y = rnd((6,), 1, 7), rnd((5,), 2, 7)
    A = np.outer(x, y)
    B = np.outer(y, x)
    s = O.scalar(A, "ia", B, "ai", 0.5)
    assert abs(s - 0.5 * float(x @ x) * float(y @ y)) < 1e-14 * abs(s)
    no, nv = 4, 6
    rng = np.random.default_rng(1)
    eo = np.sort(rng.uniform(-2, -1, no))
    ev = np.sort(rng.uniform(1, 2, nv))
    Voovv = rnd((no, no, nv, nv), 3, 4)
    D = eo[:, None, None, None] + eo[None, :, None, None] - ev[None, None, :, None] - ev[None, None, None, :]
    T2 = Voovv / D
    E = O.scalar(Voovv, "ijab", T2, "ijab", 0.25)
    assert E < 0


def test_antisymmetry_preserved():
    """S633: antisymmetric V (a<->b, c<->d) and T (c<->d, i<->j) => ladder R antisymmetric."""
    V, Oo = 4, 3
    X = rnd((V, V, V, V), 41, 4)
    Vt = X - X.transpose(1, 0, 2, 3)
    Vt = Vt - Vt.transpose(0, 1, 3, 2)
    Y = rnd((V, V, Oo, Oo), 41, 5)
    T = Y - Y.transpose(1, 0, 2, 3)
    T = T - T.transpose(0, 1, 3, 2)
    R = O.contract(np.zeros((V, V, Oo, Oo)), "abij", Vt, "abcd", T, "cdij", 1.0, 0.0)
    assert np.abs(R + R.transpose(1, 0, 2, 3)).max() < 1e-13
    assert np.abs(R + R.transpose(0, 1, 3, 2)).max() < 1e-13


def test_masked_output_and_zero_blocks():
    """Zeros in, zeros out (S216, S730): zero C blocks untouched; zero A/B blocks read as 0."""
    so = L.IndexSpace(4, [(0, 2, 1), (2, 4, -1)])
    sv = L.IndexSpace(6, [(0, 3, 1), (3, 6, -1)])
    tO, tV = L.tile_fixed(so, 2), L.tile_fixed(sv, 3)
    Ct = L.tensor_spin([tV, tV, tO, tO], [0, 1], [2, 3])
    m = O.nz_mask(Ct)
    C = rnd(Ct.shape, 1, 3)
    A = rnd((6, 6, 4, 4), 1, 1)
    B = rnd((6, 6, 4, 4), 1, 2)
    got = O.contract(C, "abij", A, "acik", B, "cbkj", 1.0, 1.0, cmask=m)
    assert np.array_equal(got[m == 0], C[m == 0])
    ref = C + np.einsum("acik,cbkj->abij", A, B)
    assert normwise(got[m == 1], ref[m == 1]) < 1e-14


# ------------------------------------------------------------------ task list (closed forms)

def spaces(O_, V_, tO, tV, spin):
    if spin:
        so = L.IndexSpace(O_, [(0, O_ // 2, 1), (O_ // 2, O_, -1)])
        sv = L.IndexSpace(V_, [(0, V_ // 2, 1), (V_ // 2, V_, -1)])
    else:
        so, sv = L.IndexSpace(O_), L.IndexSpace(V_)
    return L.tile_fixed(so, tO), L.tile_fixed(sv, tV)


def ccsd_terms(O_, V_, tO, tV, spin):
    """Synthetic CC maps, reading R7: V{ab|cd}, T{cd|ij}, R{ab|ij}, ring A{ac|ik}, B{kb|cj}, W{kl|ij}."""
    o, v = spaces(O_, V_, tO, tV, spin)
    mk = (lambda dims, up, lo: L.tensor_spin(dims, up, lo)) if spin else (lambda dims, up, lo: L.tensor_dense_map(dims))
    R = mk([v, v, o, o], [0, 1], [2, 3])
    ladder = (R, "abij", mk([v, v, v, v], [0, 1], [2, 3]), "abcd", mk([v, v, o, o], [0, 1], [2, 3]), "cdij")
    ring = (R, "abij", mk([v, v, o, o], [0, 1], [2, 3]), "acik", mk([v, v, o, o], [2, 1], [0, 3]), "cbkj")
    hh = (R, "abij", mk([v, v, o, o], [0, 1], [2, 3]), "abkl", mk([o, o, o, o], [0, 1], [2, 3]), "klij")
    return dict(ladder=ladder, ring=ring, hh=hh)


def test_task_counts_config1_config2():
    """cfg1 ring O=4 V=8 tile 4 dense: 8 tasks; cfg2 ladder O=40 V=200 tile 40: 625 = 5^4 (App. A)."""
    t = ccsd_terms(4, 8, 4, 4, False)["ring"]
    cb, ptr, ab, bb, cost = L.task_list(*t)
    assert len(ab) == 8 and len(cb) == 4
    assert sum(cost) == 2 * 8 * 8 * 4 * 4 * 8 * 4 == 65536
    t = ccsd_terms(40, 200, 40, 40, False)["ladder"]
    cb, ptr, ab, bb, cost = L.task_list(*t)
    assert len(ab) == 625 and len(cb) == 25 and sum(cost) == 2 * 200 ** 4 * 40 ** 2


@pytest.mark.parametrize("term,count", [("ladder", 6250), ("ring", 1250), ("hh", 250)])
def test_task_counts_config3_spin(term, count):
    """cfg3 O=60 V=400 tO=30 tV=40 alpha/beta maps (reading R7, R15): 150 of 400 R blocks non-zero;
    tasks ladder 6250 / ring 1250 / hh 250; FLOPs exactly 10/64 of dense."""
    ts = ccsd_terms(60, 400, 30, 40, True)[term]
    cb, ptr, ab, bb, cost = L.task_list(*ts)
    assert len(cb) == 150 and len(ab) == count
    td = ccsd_terms(60, 400, 30, 40, False)[term]
    dense_cost = sum(L.task_list(*td)[4])
    assert sum(cost) * 64 == dense_cost * 10


def test_task_list_canonical_order_and_validity():
    """CSR by non-zero C block in row-major order; contracted tuples row-major; every task's A and
    B blocks non-zero; no task for a zero pair (S509)."""
    ts = ccsd_terms(8, 12, 2, 3, True)["ring"]
    C, c, A, a, B, b = ts
    cb, ptr, ab, bb, cost = L.task_list(*ts)
    assert cb == sorted(cb) and all(C.nz[x] for x in cb) and len(cb) == sum(C.nz)
    for i in range(len(cb)):
        seg = list(zip(ab[ptr[i]:ptr[i + 1]], bb[ptr[i]:ptr[i + 1]]))
        assert all(A.nz[x] and B.nz[y] for x, y in seg)
        # contracted labels of ring in A order: c, k -> tuple = (tile c, tile k), row-major
        keys = [(A.block_coords(x)[1], A.block_coords(x)[3]) for x, _ in seg]
        assert keys == sorted(keys)


def test_blockwise_tasks_reproduce_dense_definition():
    """The task-list decomposition (sum over non-zero pairs of per-block contractions) equals the
    dense definition on non-zero C blocks (pins the task list semantics, P111/P138/P210)."""
    ts = ccsd_terms(8, 12, 2, 3, True)["ring"]
    Ct, c, At, a, Bt, b = ts
    Cd, Ad, Bd = (O.dense_masked(T, rnd(T.shape, 9, tag)) for T, tag in ((Ct, 3), (At, 1), (Bt, 2)))
    ref = O.contract(Cd, c, Ad, a, Bd, b, 1.0, 1.0, cmask=O.nz_mask(Ct))
    cb, ptr, ab, bb, cost = L.task_list(*ts)
    out = Cd.copy()
    for i, cblk in enumerate(cb):
        csl = tuple(slice(o, o + e) for o, e in zip(Ct.block_origin(cblk), Ct.block_extents(cblk)))
        for ab_, bb_ in zip(ab[ptr[i]:ptr[i + 1]], bb[ptr[i]:ptr[i + 1]]):
            asl = tuple(slice(o, o + e) for o, e in zip(At.block_origin(ab_), At.block_extents(ab_)))
            bsl = tuple(slice(o, o + e) for o, e in zip(Bt.block_origin(bb_), Bt.block_extents(bb_)))
            out[csl] += np.einsum(f"{a},{b}->{c}", Ad[asl], Bd[bsl])
    assert normwise(out, ref) < 1e-13


def test_lpt_partition():
    """LPT: every block once; hand-worked example; makespan within the 4/3 bound of a brute-force
    optimum on a tiny instance."""
    cost = [7, 7, 6, 6, 5, 4, 4, 2]
    ids = list(range(8))
    own = L.lpt_partition(cost, ids, 3)
    # by hand, (cost desc, id asc), least-loaded rank, ties lowest:
    # 7->r0 (7,0,0); 7->r1 (7,7,0); 6->r2 (7,7,6); 6->r2 (7,7,12); 5->r0 (12,7,12);
    # 4->r1 (12,11,12); 4->r1 (12,15,12); 2->r0 (14,15,12)
    assert own == [0, 1, 2, 2, 0, 1, 1, 0]
    loads = [sum(c for c, o in zip(cost, own) if o == r) for r in range(3)]
    assert loads == [14, 15, 12]
    best = min(max(sum(c for c, o in zip(cost, asg) if o == r) for r in range(3))
               for asg in product(range(3), repeat=8))
    assert max(loads) <= (4 / 3 - 1 / 9) * best + 1e-9


def test_sampled_elements_match_full():
    """Sampled-element oracle (used at full bench sizes) == full oracle on a small case."""
    c, a, b, ext = CASES[0]
    sh = lambda s: tuple(ext[x] for x in s)
    A = rnd(sh(a), 4, 1)
    B = rnd(sh(b), 4, 2)
    full = O.contract(np.zeros(sh(c)), c, A, a, B, b, 1.0, 0.0)
    idx = np.array([[0, 0, 0, 0], [4, 3, 2, 1], [2, 1, 0, 1]])
    got = O.sampled_elements(idx, c, a, b, ext,
                             lambda ix: S.values(4, 1, S.linear_index(sh(a), ix)),
                             lambda ix: S.values(4, 2, S.linear_index(sh(b), ix)))
    assert np.array_equal(got, full[tuple(idx.T)])


def test_cholesky_v_pins():
    """Eq. cc12 oracle: brute force on a tiny case, antisymmetry (p<->q, r<->s), closed forms:
    separable rank-1 X gives V = 0; X(p,r,L) = delta_pr delta_L0 gives V = d_pr d_qs - d_ps d_qr."""
    n, nl = 4, 3
    X = rnd((n, n, nl), 5, 7)
    V = O.cholesky_v(X)
    for p, q, r, s in [(0, 1, 2, 3), (3, 3, 1, 0), (2, 0, 2, 1)]:
        bf = sum(X[p, r, l] * X[q, s, l] - X[p, s, l] * X[q, r, l] for l in range(nl))
        assert abs(V[p, q, r, s] - bf) < 1e-15
    assert np.abs(V + V.transpose(1, 0, 2, 3)).max() < 1e-15
    assert np.abs(V + V.transpose(0, 1, 3, 2)).max() < 1e-15
    x, y, z = rnd((n,), 1, 7), rnd((n,), 2, 7), rnd((nl,), 3, 7)
    X1 = np.einsum("p,r,l->prl", x, y, z)
    assert np.abs(O.cholesky_v(X1)).max() < 1e-15
    Xd = np.zeros((n, n, nl))
    Xd[np.arange(n), np.arange(n), 0] = 1.0
    I = np.eye(n)
    assert np.array_equal(O.cholesky_v(Xd), np.einsum("pr,qs->pqrs", I, I) - np.einsum("ps,qr->pqrs", I, I))


def test_cholesky_v_row_and_ladder_sample_pins():
    """Row form of Eq. cc12 (sampled checks at configs[4] scale): brute force per element, closed
    forms (separable X: 0; X(p,r,L) = delta_pr delta_L0: d_ar d_bs - d_as d_br), antisymmetry in
    (r,s); the ladder sample is the brute-force double sum."""
    n, nl = 5, 4
    X = rnd((n, n, nl), 6, 7)
    for a, b in [(0, 1), (3, 3), (4, 2)]:
        v = O.cholesky_v_row(X[a], X[b])
        for r in range(n):
            for s in range(n):
                bf = sum(X[a, r, l] * X[b, s, l] - X[a, s, l] * X[b, r, l] for l in range(nl))
                assert abs(v[r, s] - bf) < 1e-15
        assert np.abs(v + v.T).max() < 1e-15
    x, y, z = rnd((n,), 1, 8), rnd((n,), 2, 8), rnd((nl,), 3, 8)
    X1 = np.einsum("p,r,l->prl", x, y, z)
    assert np.abs(O.cholesky_v_row(X1[1], X1[3])).max() < 1e-15
    Xd = np.zeros((n, n, nl))
    Xd[np.arange(n), np.arange(n), 0] = 1.0
    I = np.eye(n)
    assert np.array_equal(O.cholesky_v_row(Xd[1], Xd[3]), np.outer(I[1], I[3]) - np.outer(I[3], I[1]))
    T = rnd((n, n), 4, 8)
    v = O.cholesky_v_row(X[2], X[0])
    bf = 0.0
    for r in range(n):
        for s in range(n):
            bf += v[r, s] * T[r, s]
    assert abs(O.ladder_sample(v, T, 0.5) - 0.5 * bf) < 1e-14


def test_freivalds_pins():
    """Freivalds check: exact results give a residual at rounding level for a permuted-label ring
    term; one perturbed element of C (1e-9 relative) is detected for random x; the right side is the
    brute-force vector sum."""
    rng = np.random.default_rng(3)
    ext = dict(a=5, b=4, c=3, i=2, j=3, k=4)
    A = rnd((ext["a"], ext["c"], ext["i"], ext["k"]), 7, 9)         # A(a,c,i,k)
    B = rnd((ext["c"], ext["b"], ext["k"], ext["j"]), 8, 9)         # B(c,b,k,j)
    C0 = rnd((ext["a"], ext["b"], ext["i"], ext["j"]), 9, 9)
    C = O.contract(C0.copy(), "abij", A, "acik", B, "cbkj", 0.7, 1.3)
    x = rng.uniform(-1, 1, (ext["b"], ext["j"]))
    lhs, rhs = O.freivalds(C, "abij", A, "acik", B, "cbkj", x, 0.7, 1.3, C0)
    assert np.abs(lhs - rhs).max() <= 1e-13 * np.abs(lhs).max()
    bf = np.zeros((ext["a"], ext["i"]))
    for a in range(ext["a"]):
        for i in range(ext["i"]):
            s = 0.0
            for b in range(ext["b"]):
                for j in range(ext["j"]):
                    t = 1.3 * C0[a, b, i, j]
                    for c in range(ext["c"]):
                        for k in range(ext["k"]):
                            t += 0.7 * A[a, c, i, k] * B[c, b, k, j]
                    s += t * x[b, j]
            bf[a, i] = s
    assert np.abs(rhs - bf).max() <= 1e-13 * np.abs(bf).max()
    Cbad = C.copy()
    Cbad[2, 1, 0, 2] *= 1 + 1e-9
    lhs2, _ = O.freivalds(Cbad, "abij", A, "acik", B, "cbkj", x, 0.7, 1.3, C0)
    assert np.abs(lhs2 - rhs).max() > 1e-11 * np.abs(C).max()


# ------------------------------------------------------------------ add / scalar under k-cycle label maps

def _brute_permuted(A, a_lbl, c_lbl):
    """Pure-Python definition of P173 ``C(c_lbl) = A(a_lbl)``: C[x] = A[x re-indexed by label]."""
    shape = tuple(A.shape[a_lbl.index(l)] for l in c_lbl)
    C = np.empty(shape)
    for x in product(*[range(n) for n in shape]):
        lab = dict(zip(c_lbl, x))
        C[x] = A[tuple(lab[l] for l in a_lbl)]
    return C


# (c_lbl, a_lbl): 2-cycles, 3-cycles and 4-cycles of the label map, with distinct
# extents per label so that any inverted / transposed map changes shapes or values
K_CYCLES = [("abij", "bija"), ("abij", "jabi"), ("abij", "ijab"), ("abij", "baji"), ("abc", "cab"),
            ("abc", "bca"), ("ia", "ai"), ("abij", "ajbi"), ("abij", "aijb")]


@pytest.mark.parametrize("c_lbl,a_lbl", K_CYCLES)
def test_add_k_cycles_vs_einsum_and_brute_force(c_lbl, a_lbl):
    """P173 AddOp 'with respect to the label permutation': ops.add equals numpy.einsum (independent
    library routine) and the pure-Python element loop, for beta in {0, 1, -0.5}."""
    ext = {"a": 3, "b": 4, "c": 2, "i": 5, "j": 2}
    A = rnd(tuple(ext[l] for l in a_lbl), 41, 1)
    C0 = rnd(tuple(ext[l] for l in c_lbl), 41, 3)
    perm_ref = np.einsum(f"{a_lbl}->{c_lbl}", A)
    assert np.array_equal(perm_ref, _brute_permuted(A, a_lbl, c_lbl))
    for beta in (0.0, 1.0, -0.5):
        got = O.add(C0, c_lbl, A, a_lbl, 0.75, beta)
        ref = 0.75 * perm_ref if beta == 0.0 else beta * C0 + 0.75 * perm_ref
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("c_lbl,a_lbl", K_CYCLES)
def test_scalar_k_cycles_vs_brute_force(c_lbl, a_lbl):
    """Order-0 contraction s = alpha * sum_x A[x_A] B[x_B]: ops.scalar equals a pure-Python loop over
    the label values (exact on integer inputs), and numpy.einsum on uniform inputs."""
    ext = {"a": 3, "b": 4, "c": 2, "i": 5, "j": 2}
    for kind in (S.KIND_INTEGER, S.KIND_UNIFORM):
        A = rnd(tuple(ext[l] for l in a_lbl), 43, 1, kind)
        B = rnd(tuple(ext[l] for l in c_lbl), 43, 2, kind)
        s = O.scalar(A, a_lbl, B, c_lbl, -0.5)
        if kind == S.KIND_INTEGER:
            tot = 0.0
            for x in product(*[range(ext[l]) for l in c_lbl]):
                lab = dict(zip(c_lbl, x))
                tot += A[tuple(lab[l] for l in a_lbl)] * B[x]
            assert s == -0.5 * tot
        else:
            ref = -0.5 * float(np.einsum(f"{a_lbl},{c_lbl}->", A, B))
            assert abs(s - ref) <= 1e-14 * max(abs(ref), 1.0)


def test_add_inverse_cycle_is_detected():
    """A 3-cycle and its inverse differ: the pins above would fail an inverted permutation."""
    X = rnd((3, 3, 3), 45, 1)
    assert not np.array_equal(O.add(X, "abc", X, "cab", 1.0, 0.0), O.add(X, "abc", X, "bca", 1.0, 0.0))
