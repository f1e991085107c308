"""intermediate factorization (PAPER Eqs. cc9-cc11, P293-311) and sub-space slicing
(P116-122, P152, P159).

CPU part (no GPU): the oracle pinned against things other than itself (pure-Python brute force, exact
associativity on integer inputs, the paper's cost classes n_o^4 n_u^4 vs n_o^4 n_u^2 as closed forms,
Fig. 2 sub-spaces, slice additivity), and libtt's host planning compared bit for bit with the oracle.
GPU part: tt_contract3 and sliced views against the oracle on seeded inputs (normwise <= 1e-11, R13).
"""
import itertools

import numpy as np
import pytest

import synthetic as S
from oracle import layout as L
from oracle import ops as O
from tests.cases import SpaceSpec, TensorSpec, Problem, oracle_objects, product_objects

TOL = 1e-11


def cc9_problem(O_, V_, tO, tV, spin):
    """cc9: R(a,b,i,j) += 1/4 v(e,f,m,n) t(e,f,i,j) t(a,b,m,n) (v^{ef}_{mn} stored as v(e,f,m,n))."""
    spaces = {"O": SpaceSpec(O_, tile=tO, spin_split=spin), "V": SpaceSpec(V_, tile=tV, spin_split=spin)}
    ls = {x: "V" for x in "abef"}
    ls.update({x: "O" for x in "ijmn"})
    sp = (lambda up, lo: ("spin", up, lo)) if spin else (lambda up, lo: None)
    tensors = {"R": TensorSpec("abij", sp([0, 1], [2, 3])), "v": TensorSpec("efmn", sp([0, 1], [2, 3])),
               "t": TensorSpec("efij", sp([0, 1], [2, 3]))}
    return Problem(spaces, ls, tensors)


# ------------------------------------------------------------------------------------------ oracle pins

def test_contract3_naive_vs_python_brute_force():
    rng = np.random.default_rng(3)
    nO, nV = 2, 3
    v = rng.uniform(-1, 1, (nV, nV, nO, nO))
    t1 = rng.uniform(-1, 1, (nV, nV, nO, nO))
    t2 = rng.uniform(-1, 1, (nV, nV, nO, nO))
    R = rng.uniform(-1, 1, (nV, nV, nO, nO))
    got = O.contract3_naive(R, "abij", v, "efmn", t1, "efij", t2, "abmn", 0.25, 0.5)
    ref = np.empty_like(R)
    for a, b, i, j in itertools.product(range(nV), range(nV), range(nO), range(nO)):
        s = 0.0
        for e, f, m, n in itertools.product(range(nV), range(nV), range(nO), range(nO)):
            s = s + (v[e, f, m, n] * t1[e, f, i, j]) * t2[a, b, m, n]
        ref[a, b, i, j] = 0.5 * R[a, b, i, j] + 0.25 * s
    assert np.array_equal(got, ref)   # same products, same order: bit for bit


def test_contract3_naive_equals_factorized_exactly_on_integers():
    """Eqs. cc10/cc11 reach exactly the cc9 value: with integer inputs every partial sum is exact, so the
    naive loop and the two binary oracle contractions must agree bit for bit."""
    sh = (4, 4, 3, 3)
    v, t = (S.dense(sh, 1, tag, S.KIND_INTEGER) for tag in (6, 5))
    R0 = np.zeros(sh)
    naive = O.contract3_naive(R0, "abij", v, "efmn", t, "efij", t, "abmn", 1.0, 0.0)
    I = O.contract(np.zeros((3, 3, 3, 3)), "mnij", v, "efmn", t, "efij", 1.0, 0.0)
    fact = O.contract(R0, "abij", I, "mnij", t, "abmn", 1.0, 0.0)
    assert np.array_equal(naive, fact)
    assert np.abs(naive).max() > 0


def test_contract3_rank1_closed_form():
    """v = x_e x_f y_m y_n, t = p_e p_f q_i q_j  =>  sum v t t = (x.p)^2 (y.u)^2 q_i q_j w_a w_b  (t2 = w w u u)."""
    rng = np.random.default_rng(7)
    x, p, w = (rng.uniform(-1, 1, 5) for _ in range(3))
    y, q, u = (rng.uniform(-1, 1, 3) for _ in range(3))
    v = np.einsum("e,f,m,n->efmn", x, x, y, y)
    t1 = np.einsum("e,f,i,j->efij", p, p, q, q)
    t2 = np.einsum("a,b,m,n->abmn", w, w, u, u)
    got = O.contract3_naive(np.zeros((5, 5, 3, 3)), "abij", v, "efmn", t1, "efij", t2, "abmn", 1.0, 0.0)
    ref = np.einsum("a,b,i,j->abij", w, w, q, q) * (x @ p) ** 2 * (y @ u) ** 2
    assert np.abs(got - ref).max() <= 1e-14 * np.abs(ref).max()


@pytest.mark.parametrize("nO,nV,tO,tV", [(8, 16, 4, 4), (6, 10, 3, 5), (4, 12, 4, 6)])
def test_contract3_plan_cost_classes(nO, nV, tO, tV):
    """P299 vs P311 (S577): naive n_o^4 n_u^4 multiply-adds; the cc10/cc11 factorization costs two GEMM
    passes of n_o^4 n_u^2 each (FLOPs = 2 x multiply-adds); the other pairings cost n_o^2 n_u^4 twice
    and (outer product then full contraction) n_o^4 n_u^4 twice."""
    orc = oracle_objects(cc9_problem(nO, nV, tO, tV, False))
    plan = L.contract3_plan(orc["R"], "abij", orc["v"], "efmn", orc["t"], "efij", orc["t"], "abmn")
    assert plan["naive_macs"] == nO ** 4 * nV ** 4
    assert plan["flops"] == [4.0 * nO ** 4 * nV ** 2, 4.0 * nO ** 2 * nV ** 4, 4.0 * nO ** 4 * nV ** 4]
    assert plan["pair"] == (0 if nO < nV else 1) and plan["i_lbl"] == "mnij"


def test_tile_sub_fig2():
    """Fig. 2 (P117-127): K{range(20), "first" [0,10), "second" [10,20)}, tK{K,5}; tK("first") has two
    tiles of 5 (P152); sub-spaces must sit on tile boundaries."""
    K = L.IndexSpace(20, [(0, 10, 0), (10, 20, 0)])
    tK = L.tile_fixed(K, 5)
    f, s = L.tile_range(tK, 0), L.tile_range(tK, 1)
    assert f.offsets == [0, 5, 10] and s.offsets == [0, 5, 10]
    assert L.tile_sub(tK, 5, 20).offsets == [0, 5, 10, 15]
    with pytest.raises(L.OracleError):
        L.tile_sub(tK, 3, 10)


def test_slices_partition_the_contraction():
    """P159: an operation over sub-space labels acts on the slice.  Contracting over "first" plus over
    "second" equals contracting over the whole space (a wrong slice offset breaks this), and with
    A = 1, B = -1 (Fig. 5 values) each half gives -10 against -20 for the whole."""
    A = S.dense((30, 20), 1, 1)
    B = S.dense((20, 100), 1, 2)
    full = O.contract(np.zeros((30, 100)), "ia", A, "il", B, "la", 1.0, 0.0)
    halves = np.zeros((30, 100))
    for r in ((0, 10), (10, 20)):
        halves = O.contract(halves, "ia", O.slice_of(A, [(0, 30), r]), "ix", O.slice_of(B, [r, (0, 100)]), "xa",
                            1.0, 1.0)
    assert np.abs(halves - full).max() <= 1e-14 * np.abs(full).max()
    ones = O.contract(np.zeros((30, 100)), "ia", np.ones((30, 10)), "ix", -np.ones((10, 100)), "xa", 1.0, 0.0)
    assert np.all(ones == -10.0)


# ------------------------------------------------------------------------------------ host ABI vs oracle

@pytest.fixture(scope="module")
def tt():
    import paper_2201_01257_b200 as m
    return m


@pytest.mark.parametrize("spin", [False, True])
@pytest.mark.parametrize("shape", [(8, 16, 4, 4), (6, 10, 3, 5), (8, 12, 2, 3)])
def test_contract3_plan_matches_oracle(tt, spin, shape):
    pb = cc9_problem(*shape, spin)
    orc = oracle_objects(pb)
    ctx = tt.Context(device=-1)
    P = product_objects(tt, ctx, pb)
    for args in (("abij", "efmn", "efij", "abmn"), ("abij", "abmn", "efmn", "efij"), ("abij", "efij", "abmn", "efmn")):
        cl, l1, l2, l3 = args
        ops = {"efmn": "v", "efij": "t", "abmn": "t"}
        got = tt.contract3(ctx, P["R"], cl, 1.0, 0.25, P[ops[l1]], l1, P[ops[l2]], l2, P[ops[l3]], l3)
        ref = L.contract3_plan(orc["R"], cl, orc[ops[l1]], l1, orc[ops[l2]], l2, orc[ops[l3]], l3)
        assert got["pair"] == ref["pair"] and got["i_lbl"] == ref["i_lbl"]
        assert got["flops"] == ref["flops"] and got["naive_macs"] == ref["naive_macs"]


def test_contract3_label_errors(tt):
    pb = cc9_problem(4, 8, 2, 4, False)
    ctx = tt.Context(device=-1)
    P = product_objects(tt, ctx, pb)
    with pytest.raises(tt.TTError) as e:
        tt.contract3(ctx, P["R"], "abij", 1.0, 1.0, P["v"], "abmn", P["t"], "efij", P["t"], "abmn")
    assert e.value.name == "TT_E_LABEL"


def test_subspace_and_view_layout(tt):
    ctx = tt.Context(device=-1)
    K = tt.IndexSpace(20, [(0, 10), (10, 20)], names=["first", "second"])
    tK = tt.TiledIndexSpace(K, 5)
    M = tt.IndexSpace(30)
    tM = tt.TiledIndexSpace(M, sizes=[10, 20])
    assert list(tK("first").offsets) == [0, 5, 10] and list(tK("second").offsets) == [0, 5, 10]
    assert list(tK.sub(5, 20).offsets) == [0, 5, 10, 15]
    with pytest.raises(tt.TTError) as e:
        tK.sub(3, 10)
    assert e.value.name == "TT_E_TILING"
    A = tt.Tensor(ctx, [tM, tK])             # Fig. 2: a 30 x 20 matrix with eight blocks (P140)
    assert A.nblocks == 8
    # oracle layout of the parent, restricted to the shifted tiles
    oK = L.tile_fixed(L.IndexSpace(20, [(0, 10, 0), (10, 20, 0)]), 5)
    oA = L.tensor_dense_map([L.tile_custom(L.IndexSpace(30), [10, 20]), oK])
    off = oA.blk_off()
    sub = tK("second")
    V = A.view([tM, sub])
    assert V.shape == (30, 10) and V.nblocks == 4
    assert list(V.blk_off) == [off[oA.block_id([m, 2 + k])] for m in range(2) for k in range(2)]
    with pytest.raises(tt.TTError) as e:
        A.view([tM, tt.TiledIndexSpace(K, 5)])   # not a sub-space of A's dim
    assert e.value.name == "TT_E_TILING"
    with pytest.raises(tt.TTError) as e:
        V.set_owner(np.zeros(4, np.int32))
    assert e.value.name == "TT_E_UNSUPPORTED"


# ------------------------------------------------------------------------------------------- GPU parity

@pytest.fixture(scope="module")
def gpu():
    import torch
    import paper_2201_01257_b200 as m
    torch.cuda.init()
    return m, torch


def _ctx(m, torch):
    return m.Context(device=0, stream=torch.cuda.current_stream().cuda_stream)


@pytest.mark.gpu
@pytest.mark.parametrize("spin,shape", [(False, (8, 16, 4, 4)), (True, (12, 20, 3, 5)), (False, (7, 13, 3, 5))])
def test_contract3_gpu_parity(gpu, spin, shape):
    m, torch = gpu
    pb = cc9_problem(*shape, spin)
    orc = oracle_objects(pb)
    ctx = _ctx(m, torch)
    P = product_objects(tt=m, ctx=ctx, pb=pb)
    dense, keep = {}, []
    for name, tag in (("R", 3), ("v", 6), ("t", 5)):
        dense[name] = O.dense_masked(orc[name], S.dense(orc[name].shape, 2, tag))
        buf = torch.from_numpy(O.pack(orc[name], dense[name])).cuda()
        P[name].bind(buf)
        keep.append(buf)
    plan = m.contract3(ctx, P["R"], "abij", 0.5, 0.25, P["v"], "efmn", P["t"], "efij", P["t"], "abmn")
    ws = torch.empty(plan["ws_elems"], dtype=torch.float64, device="cuda")
    info = m.contract3(ctx, P["R"], "abij", 0.5, 0.25, P["v"], "efmn", P["t"], "efij", P["t"], "abmn", ws)
    got = P["R"].download()
    ctx.sync()
    ref = O.contract3_naive(dense["R"], "abij", dense["v"], "efmn", dense["t"], "efij", dense["t"], "abmn", 0.25,
                            0.5, cmask=O.nz_mask(orc["R"]))
    ref = O.pack(orc["R"], ref)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err <= TOL, err
    assert info["pair"] == 0 and info["i_lbl"] == "mnij"
    st = ctx.stats()
    assert st["flops"] == info["flops"][0]


@pytest.mark.gpu
def test_views_gpu_parity(gpu):
    """Sliced operands and a sliced output (P152, P159): C(i, a in "second") += A(i, x in "first") B(x, a),
    then an add into a slice; the untouched part of C must be unchanged bit for bit."""
    m, torch = gpu
    ctx = _ctx(m, torch)
    K = m.IndexSpace(40, [(0, 16), (16, 40)], names=["first", "second"])
    tK = m.TiledIndexSpace(K, 8)
    M = m.IndexSpace(30)
    tM = m.TiledIndexSpace(M, sizes=[10, 20])
    N = m.IndexSpace(40, [(0, 16), (16, 40)], names=["first", "second"])
    tN = m.TiledIndexSpace(N, 8)
    A, B, C = m.Tensor(ctx, [tM, tK]), m.Tensor(ctx, [tK, tN]), m.Tensor(ctx, [tM, tN])
    oK = L.tile_fixed(L.IndexSpace(40, [(0, 16, 0), (16, 40, 0)]), 8)
    oM = L.tile_custom(L.IndexSpace(30), [10, 20])
    oA, oB, oC = L.tensor_dense_map([oM, oK]), L.tensor_dense_map([oK, oK]), L.tensor_dense_map([oM, oK])
    DA, DB, DC = S.dense((30, 40), 3, 1), S.dense((40, 40), 3, 2), S.dense((30, 40), 3, 3)
    bufs = []
    for T, oT, D in ((A, oA, DA), (B, oB, DB), (C, oC, DC)):
        b = torch.from_numpy(O.pack(oT, D)).cuda()
        T.bind(b)
        bufs.append(b)
    Cv = C.view([tM, tN("second")])
    m.contract(ctx, Cv, "ia", 1.0, 0.5, A.view([tM, tK("first")]), "ix", B.view([tK("first"), tN("second")]), "xa")
    m.add(ctx, Cv, "ia", 1.0, -2.0, A.view([tM, tK("second")]), "ia")
    got = O.unpack(oC, C.download())
    ctx.sync()
    ref = DC.copy()
    sec, fst = (16, 40), (0, 16)
    cs = O.slice_of(ref, [(0, 30), sec])
    cs[...] = O.contract(cs, "ia", O.slice_of(DA, [(0, 30), fst]), "ix", O.slice_of(DB, [fst, sec]), "xa", 0.5, 1.0)
    cs[...] = O.add(cs, "ia", O.slice_of(DA, [(0, 30), sec]), "ia", -2.0, 1.0)
    assert np.array_equal(got[:, :16], DC[:, :16])
    assert np.abs(got - ref).max() / np.abs(ref).max() <= TOL


def test_parent_layout_frozen_while_views_live(tt):
    """A view captures its parent's block map, offsets and owners (R29): while it lives, ownership /
    compact / partition changes of the parent are refused (TT_E_STATE) instead of leaving the view
    stale; after the view is destroyed they succeed."""
    ctx = tt.Context(device=-1, rank=0, nranks=2)
    M, K = tt.IndexSpace(30), tt.IndexSpace(20, [(0, 10), (10, 20)], names=["first", "second"])
    tM, tK = tt.TiledIndexSpace(M, sizes=[10, 20]), tt.TiledIndexSpace(K, 5)
    A = tt.Tensor(ctx, [tM, tK])
    V = A.view([tM, tK("first")])
    for fn in (lambda: A.set_owner([1] * A.nblocks), lambda: A.set_compact(True),
               lambda: A.set_parts([(0, 0, 5, 0), (0, 5, 10, 1)])):
        with pytest.raises(tt.TTError) as e:
            fn()
        assert e.value.name == "TT_E_STATE"
    V.close()
    A.set_owner([1] * A.nblocks)
    assert list(A.owner) == [1] * A.nblocks
