"""CPU tests of libtt's host side through the C ABI (host-only context, no GPU needed):
symbol exports, tilings and tile maps (bit-exact vs the oracle), validation errors, the host task
list and LPT partition (bit-exact vs the oracle enumerator), gather plans."""
import os
import re

import numpy as np
import pytest

import paper_2201_01257_b200 as tt
from oracle import layout as L
from tests.cases import Problem, SpaceSpec, TensorSpec, ccsd_problem, oracle_objects, product_objects

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hctx():
    c = tt.Context(device=-1)
    yield c
    c.close()


def test_exports_every_declared_symbol():
    """Every function declared in include/tt.h is exported by libtt.so and bound by the wrapper."""
    hdr = open(os.path.join(ROOT, "include", "tt.h")).read()
    declared = set(re.findall(r"^(?:tt_status|const char\*|int32_t)\s+(tt_\w+)\(", hdr, re.M))
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(tt._lib, name), name
    assert declared == set(tt.EXPORTED)


def test_fig2_layout(hctx):
    """P140: A{tM,tK} 30x20 with eight blocks; packed offsets = oracle (bit-exact)."""
    N, M, K = tt.IndexSpace(100), tt.IndexSpace(30), tt.IndexSpace(20)
    tN, tM, tK = tt.TiledIndexSpace(N, 10), tt.TiledIndexSpace(M, sizes=[10, 20]), tt.TiledIndexSpace(K, 5)
    assert tN.ntiles == 10 and tK.ntiles == 4 and list(tM.offsets) == [0, 10, 30]
    A = tt.Tensor(hctx, [tM, tK])
    assert A.nblocks == 8 and A.shape == (30, 20)
    oA = L.tensor_dense_map([L.tile_custom(L.IndexSpace(30), [10, 20]), L.tile_fixed(L.IndexSpace(20), 5)])
    assert list(A.blk_off) == oA.blk_off() and A.packed_elems == oA.packed_elems()


def test_tiling_errors():
    K = tt.IndexSpace(20)
    with pytest.raises(tt.TTError) as e:
        tt.TiledIndexSpace(K, sizes=[10, 5])
    assert e.value.name == "TT_E_COVERAGE"
    sp = tt.IndexSpace(150, [(0, 75), (75, 150)], [1, -1])
    t = tt.TiledIndexSpace(sp, 64)
    assert list(np.diff(t.offsets)) == [64, 11, 64, 11] and list(t.spin) == [1, 1, -1, -1]
    with pytest.raises(tt.TTError) as e:
        tt.TiledIndexSpace(sp, sizes=[70, 80])
    assert e.value.name == "TT_E_TILING"
    with pytest.raises(tt.TTError) as e:
        tt.IndexSpace(10, [(0, 4), (5, 10)], [1, -1])
    assert e.value.name == "TT_E_COVERAGE"
    with pytest.raises(tt.TTError):
        tt.TiledIndexSpace(K, 0)


LAYOUT_PROBLEMS = [
    ccsd_problem(8, 12, 2, 3, True),
    ccsd_problem(7, 11, 3, 4, False),
    ccsd_problem(60, 400, 30, 40, True, terms=("ladder",)),
    Problem({"X": SpaceSpec(13, sizes=[5, 1, 7]), "Y": SpaceSpec(9, tile=4, spin_split=True)},
            {"p": "X", "q": "Y", "r": "X", "s": "Y"},
            {"A": TensorSpec("pqs", ("spin", [1], [2])), "B": TensorSpec("sr", ("nz", [1, 0, 1, 1, 0, 1, 0, 1, 1])),
             "C": TensorSpec("pqr", None)}),
]


@pytest.mark.parametrize("pi", range(len(LAYOUT_PROBLEMS)))
def test_tile_maps_bit_exact(hctx, pi):
    """nz maps, packed offsets (16-B aligned, R10), default RR owners (P210) == oracle."""
    pb = LAYOUT_PROBLEMS[pi]
    orc = oracle_objects(pb)
    prod = product_objects(tt, hctx, pb)
    for name in pb.tensors:
        o, p = orc[name], prod[name]
        assert list(p.nz) == o.nz, name
        assert list(p.blk_off) == o.blk_off(), name
        assert p.packed_elems == o.packed_elems(), name
        assert list(p.owner) == o.owners(), name


def test_owner_rr_multi_rank():
    c = tt.Context(device=-1, rank=1, nranks=3)
    pb = ccsd_problem(8, 12, 2, 3, True, terms=("ladder",))
    orc = oracle_objects(pb, nranks=3)
    prod = product_objects(tt, c, pb)
    assert list(prod["Vv"].owner) == orc["Vv"].owners()


def test_validation_errors(hctx):
    pb = ccsd_problem(4, 8, 4, 4, False, terms=("ring",))
    P = product_objects(tt, hctx, pb)
    R, A, B = P["R"], P["Ta"], P["Wr"]
    cases = [
        (("abij", "acik", "cbkk"), "TT_E_LABEL"),     # repeated label (S412)
        (("abij", "acik", "cbkx"), "TT_E_LABEL"),     # dangling
        (("abi", "acik", "cbkj"), "TT_E_LABEL"),      # arity
        (("abij", "abik", "cbkj"), "TT_E_LABEL"),     # b in C, A and B (batch, S380)
        (("abij", "acik", "kbcj"), "TT_E_TILING"),    # k bound to V on B, O on A (S413)
    ]
    for (cl, al, bl), err in cases:
        with pytest.raises(tt.TTError) as e:
            tt.task_list(hctx, R, cl, A, al, B, bl)
        assert e.value.name == err, (cl, al, bl)
    with pytest.raises(tt.TTError) as e:
        tt.contract(hctx, R, "abij", 1.0, 1.0, A, "acik", B, "cbkj")
    assert e.value.name == "TT_E_STATE"


TL_PROBLEMS = [ccsd_problem(4, 8, 4, 4, False), ccsd_problem(8, 12, 2, 3, True), ccsd_problem(10, 14, 3, 4, True),
               ccsd_problem(9, 13, 4, 5, False)]


@pytest.mark.parametrize("pi", range(len(TL_PROBLEMS)))
def test_host_task_list_bit_exact(hctx, pi):
    """Host enumerator == oracle brute force: C blocks, CSR, (A,B) block ids, FLOP cost (R11)."""
    pb = TL_PROBLEMS[pi]
    orc = oracle_objects(pb)
    prod = product_objects(tt, hctx, pb)
    for (c, cl, a, al, b, bl) in pb.ops:
        ocb, optr, oab, obb, ocost = L.task_list(orc[c], cl, orc[a], al, orc[b], bl)
        tl = tt.task_list(hctx, prod[c], cl, prod[a], al, prod[b], bl)
        assert list(tl["cblk"]) == ocb and list(tl["ptr"]) == optr
        assert list(tl["a_blk"]) == oab and list(tl["b_blk"]) == obb
        assert list(tl["cost"]) == ocost


def test_task_counts_closed_forms(hctx):
    """cfg2 ladder 625 tasks; cfg3 ladder/ring/hh 6250/1250/250; cfg4 ladder 40960."""
    pb = ccsd_problem(40, 200, 40, 40, False, terms=("ladder",))
    P = product_objects(tt, hctx, pb)
    assert len(tt.task_list(hctx, P["R"], "abij", P["Vv"], "abcd", P["T"], "cdij")["a_blk"]) == 625
    pb = ccsd_problem(60, 400, 30, 40, True)
    P = product_objects(tt, hctx, pb)
    got = [len(tt.task_list(hctx, P[c], cl, P[a], al, P[b], bl)["a_blk"]) for (c, cl, a, al, b, bl) in pb.ops]
    assert got == [6250, 1250, 250]
    pb = ccsd_problem(100, 800, 50, 50, True, terms=("ladder",))
    P = product_objects(tt, hctx, pb)
    tl = tt.task_list(hctx, P["R"], "abij", P["Vv"], "abcd", P["T"], "cdij")
    assert len(tl["a_blk"]) == 40960 and int(tl["cost"].sum()) == 1280000000000000


@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_lpt_partition_matches_oracle(nranks):
    c = tt.Context(device=-1, nranks=nranks)
    pb = ccsd_problem(10, 14, 3, 4, True)
    orc = oracle_objects(pb, nranks)
    prod = product_objects(tt, c, pb)
    for (C, cl, a, al, b, bl) in pb.ops:
        ocb, _, _, _, ocost = L.task_list(orc[C], cl, orc[a], al, orc[b], bl)
        oown = L.lpt_partition(ocost, ocb, nranks)
        own = tt.partition_lpt(c, prod[C], cl, prod[a], al, prod[b], bl)
        assert [own[x] for x in ocb] == oown
        assert all(own[x] == -1 for x in range(prod[C].nblocks) if not prod[C].nz[x])


def _ranges_of(T, blk, rank):
    """element ranges of block blk of product tensor T held by rank (whole / replicated / parts)."""
    vol = int(np.prod([d.offsets[t + 1] - d.offsets[t] for d, t in zip(T.dims, np.unravel_index(blk, T.grid))]))
    parts = [p for p in T.parts if p[0] == blk]
    if not parts:
        return [(0, vol)] if T.owner[blk] in (rank, tt.TT_REPLICATED) else []
    inner = vol // (parts[-1][2])
    return [(lo * inner, hi * inner) for (_, lo, hi, o) in parts if o == rank]


def _pieces(T, blk, e0, e1):
    vol = int(np.prod([d.offsets[t + 1] - d.offsets[t] for d, t in zip(T.dims, np.unravel_index(blk, T.grid))]))
    parts = [p for p in T.parts if p[0] == blk]
    if not parts:
        return [(int(T.owner[blk]), e0, e1)]
    inner = vol // parts[-1][2]
    out = []
    for (_, lo, hi, o) in parts:
        a, z = max(e0, lo * inner), min(e1, hi * inner)
        if a < z:
            out.append((o, a, z))
    return out


def _expected_gather(orc, prod, pb_op, me, nranks):
    """Needed input ranges per rank from the oracle task list and the product's ownership; the
    receives / sends of rank `me` (whole blocks, or matching rows when C is row-split along a label
    that is also the operand's dim 0)."""
    C, cl, a, al, b, bl = pb_op
    ocb, optr, oab, obb, _ = L.task_list(orc[C], cl, orc[a], al, orc[b], bl)
    need = {r: {} for r in range(nranks)}
    for g, cb in enumerate(ocb):
        cvol = orc[C].block_volume(cb)
        cin = cvol // orc[C].block_extents(cb)[0]
        for r in range(nranks):
            for (h0, h1) in _ranges_of(prod[C], cb, r):
                lo, hi = h0 // cin, h1 // cin
                for t in range(optr[g], optr[g + 1]):
                    for op, (name, lbl, blk) in enumerate(((a, al, oab[t]), (b, bl, obb[t]))):
                        vol = orc[name].block_volume(blk)
                        if lbl[0] == cl[0]:
                            inner = vol // orc[name].block_extents(blk)[0]
                            rng = (lo * inner, hi * inner)
                        else:
                            rng = (0, vol)
                        need[r].setdefault((op, blk), []).append(rng)
    recv, send = [], []
    for r in range(nranks):
        for (op, blk), rngs in need[r].items():
            rngs.sort()
            merged = []
            for x in rngs:
                if merged and x[0] <= merged[-1][1]:
                    merged[-1] = (merged[-1][0], max(merged[-1][1], x[1]))
                else:
                    merged.append(x)
            T = prod[[a, b][op]]
            for (e0, e1) in merged:
                for (src, x0, x1) in _pieces(T, blk, e0, e1):
                    if src in (tt.TT_REPLICATED, r):
                        continue
                    if r == me:
                        recv.append((op, blk, src, x0, x1))
                    if src == me:
                        send.append((op, blk, r, x0, x1))
    return sorted(recv), sorted(send)


@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("split", [False, True])
def test_gather_plan_exactly_needed_blocks(nranks, split):
    """Each rank receives exactly the A/B ranges its owned C blocks (or C row parts) read but it does
    not hold, and the sends of every rank mirror the receives of its peers (P212)."""
    pb = ccsd_problem(8, 12, 2, 3, True)
    sends, recvs = {}, {}
    for k in (0, 1):              # ladder (C dim 0 shared with A) and ring
        for me in range(nranks):
            c = tt.Context(device=-1, rank=me, nranks=nranks)
            orc = oracle_objects(pb, nranks)
            prod = product_objects(tt, c, pb)
            C, cl, a, al, b, bl = pb.ops[k]
            if split:
                tt.partition_split(c, prod[C], cl, prod[a], al, prod[b], bl)
            else:
                prod[C].set_owner(tt.partition_lpt(c, prod[C], cl, prod[a], al, prod[b], bl))
            r, s = tt.gather_plan(c, prod[C], cl, prod[a], al, prod[b], bl)
            er, es = _expected_gather(orc, prod, pb.ops[k], me, nranks)
            assert sorted(map(tuple, r.tolist())) == er
            assert sorted(map(tuple, s.tolist())) == es
            sends[me] = {(op, blk, me, peer, e0, e1) for op, blk, peer, e0, e1 in s.tolist()}
            recvs[me] = {(op, blk, peer, me, e0, e1) for op, blk, peer, e0, e1 in r.tolist()}
        assert set().union(*sends.values()) == set().union(*recvs.values())


@pytest.mark.parametrize("nranks", [2, 3, 8])
@pytest.mark.parametrize("grouped", [False, True])
def test_partition_split_matches_oracle(nranks, grouped):
    """Row-splitting water-filling partition == oracle (R24b); loads balanced to within one row."""
    c = tt.Context(device=-1, nranks=nranks)
    for pb in (ccsd_problem(40, 200, 40, 40, False, terms=("ladder",)), ccsd_problem(10, 14, 3, 4, True)):
        orc = oracle_objects(pb, nranks)
        prod = product_objects(tt, c, pb)
        C, cl, a, al, b, bl = pb.ops[0]
        ocb, _, _, _, ocost = L.task_list(orc[C], cl, orc[a], al, orc[b], bl)
        gd = (0, 1) if grouped else ()
        exp = L.partition_split(orc[C], ocost, ocb, list(gd), nranks)
        tt.partition_split(c, prod[C], cl, prod[a], al, prod[b], bl, group_dims=gd)
        got = {}
        for x in ocb:
            if prod[C].owner[x] == tt.TT_SPLIT:
                got[x] = [(lo, hi, o) for (bb, lo, hi, o) in prod[C].parts if bb == x]
            else:
                got[x] = [(0, orc[C].block_extents(x)[0], int(prod[C].owner[x]))]
        assert got == exp
        load = [0.0] * nranks
        maxrow = 0.0
        for x, cst in zip(ocb, ocost):
            rows = orc[C].block_extents(x)[0]
            maxrow = max(maxrow, cst / rows)
            for lo, hi, o in exp[x]:
                load[o] += cst * (hi - lo) / rows
        W = sum(ocost)
        tol = maxrow * (len(pb.spaces) + 4 if grouped else 1)
        assert max(load) - W / nranks <= tol + 1e-6


@pytest.mark.parametrize("nranks", [2, 5])
@pytest.mark.parametrize("grouped", [False, True])
def test_partition_split_cost_matches_oracle(nranks, grouped):
    """Caller-supplied block costs (seeded, with zeros) -> the same water-filling partition as the
    oracle's partition_split on those costs; wrong-length or negative costs are rejected."""
    c = tt.Context(device=-1, nranks=nranks)
    pb = ccsd_problem(10, 14, 3, 4, True)
    orc = oracle_objects(pb, nranks)
    prod = product_objects(tt, c, pb)
    C = pb.ops[0][0]
    cb = [int(x) for x in np.flatnonzero(orc[C].nz)]
    rng = np.random.default_rng(7)
    cost = rng.integers(0, 1000, len(cb)) * (rng.random(len(cb)) > 0.2)
    gd = (0, 1) if grouped else ()
    exp = L.partition_split(orc[C], [int(x) for x in cost], cb, list(gd), nranks)
    tt.partition_split_cost(c, prod[C], cost, group_dims=gd)
    got = {}
    for x in cb:
        if prod[C].owner[x] == tt.TT_SPLIT:
            got[x] = [(lo, hi, o) for (bb, lo, hi, o) in prod[C].parts if bb == x]
        else:
            got[x] = [(0, orc[C].block_extents(x)[0], int(prod[C].owner[x]))]
    assert got == exp
    with pytest.raises(ValueError):
        tt.partition_split_cost(c, prod[C], cost[:-1])
    bad = cost.copy()
    bad[0] = -1
    with pytest.raises(tt.TTError):
        tt.partition_split_cost(c, prod[C], bad)


@pytest.mark.parametrize("rank", [0, 1, 2])
def test_compact_storage_layout(rank):
    """Compact storage: per non-zero block the span of this rank's held ranges (owned blocks, owned
    row parts, replicated blocks) packed in block order with even (16-B aligned) bases; -1 for blocks
    not stored; recomputed on ownership changes; the global layout (tt_tensor_layout) unchanged."""
    nranks = 3
    c = tt.Context(device=-1, rank=rank, nranks=nranks)
    pb = ccsd_problem(10, 14, 3, 4, True)
    P = product_objects(tt, c, pb)
    R = P[pb.ops[0][0]]
    glob = R.blk_off.copy()
    _, cl, a, al, b, bl = pb.ops[0]
    tt.partition_split(c, R, cl, P[a], al, P[b], bl, group_dims=(0, 1))
    own = R.owner.copy()
    own[own == tt.TT_SPLIT] = 0                    # re-split by set_parts below
    rep = np.flatnonzero(R.nz)[::7]
    own[rep] = tt.TT_REPLICATED                    # some replicated blocks too (parts kept elsewhere)
    parts = [p for p in R.parts if p[0] not in set(rep.tolist())]
    R.set_owner(own)
    R.set_parts(parts)
    R.set_compact(True)
    assert np.array_equal(R.blk_off, glob)
    cur, exp = 0, np.full(R.nblocks, -1, np.int64)
    for b in range(R.nblocks):
        if not R.nz[b]:
            continue
        vol = int(np.prod([d.offsets[t + 1] - d.offsets[t] for d, t in zip(R.dims, np.unravel_index(b, R.grid))]))
        inner = vol // int(np.diff(R.dims[0].offsets)[np.unravel_index(b, R.grid)[0]])
        if R.owner[b] == rank or R.owner[b] == tt.TT_REPLICATED:
            rng = [(0, vol)]
        else:
            rng = [(lo * inner, hi * inner) for (bb, lo, hi, o) in R.parts if bb == b and o == rank]
        if not rng:
            continue
        e0, e1 = min(r[0] for r in rng), max(r[1] for r in rng)
        if (cur - e0) % 2:
            cur += 1
        exp[b] = cur - e0
        cur += e1 - e0
    assert np.array_equal(R.storage_off, exp)
    assert R.storage_elems == max(2, (cur + 1) // 2 * 2)
    assert all(x % 2 == 0 for x in R.storage_off[R.storage_off >= 0])
    R.set_compact(False)
    assert np.array_equal(R.storage_off, glob) and R.storage_elems == R.packed_elems


def test_compact_operand_cannot_receive():
    """An operand with compact storage that would have to receive remote pieces is rejected."""
    c = tt.Context(device=-1, rank=0, nranks=2)
    pb = ccsd_problem(10, 14, 3, 4, True)
    P = product_objects(tt, c, pb)
    C, cl, a, al, b, bl = pb.ops[0]
    r, _ = tt.gather_plan(c, P[C], cl, P[a], al, P[b], bl)   # A round robin: pieces received
    assert any(row[0] == 0 for row in r.tolist())
    P[a].set_compact(True)
    with pytest.raises(tt.TTError) as e:
        tt.gather_plan(c, P[C], cl, P[a], al, P[b], bl)
    assert e.value.name == "TT_E_UNSUPPORTED"
    P[a].set_owner(np.where(P[a].nz > 0, tt.TT_REPLICATED, -1).astype(np.int32))   # all local: fine
    r, s_ = tt.gather_plan(c, P[C], cl, P[a], al, P[b], bl)
    assert not any(row[0] == 0 for row in r.tolist())


@pytest.mark.parametrize("nranks", [2, 4])
def test_lpt_grouped_matches_oracle(nranks):
    """LPT over (a,b) rows of R (group dims 0,1), so each rank owns whole rows (R24)."""
    c = tt.Context(device=-1, nranks=nranks)
    pb = ccsd_problem(12, 20, 3, 4, True)
    orc = oracle_objects(pb, nranks)
    prod = product_objects(tt, c, pb)
    C, cl, a, al, b, bl = pb.ops[0]
    ocb, _, _, _, ocost = L.task_list(orc[C], cl, orc[a], al, orc[b], bl)
    oown = L.lpt_partition_grouped(orc[C], ocost, ocb, [0, 1], nranks)
    own = tt.partition_lpt(c, prod[C], cl, prod[a], al, prod[b], bl, group_dims=(0, 1))
    assert [own[x] for x in ocb] == oown
    rows = {}
    for x in ocb:
        key = orc[C].block_coords(x)[:2]
        rows.setdefault(key, set()).add(own[x])
    assert all(len(v) == 1 for v in rows.values())


def _chol_problem(tt, c, O_, V_, tO, tV, NL, tL, spin):
    so = tt.IndexSpace(O_, [(0, O_ // 2), (O_ // 2, O_)], [1, -1]) if spin else tt.IndexSpace(O_)
    sv = tt.IndexSpace(V_, [(0, V_ // 2), (V_ // 2, V_)], [1, -1]) if spin else tt.IndexSpace(V_)
    to, tv, tl = tt.TiledIndexSpace(so, tO), tt.TiledIndexSpace(sv, tV), tt.TiledIndexSpace(tt.IndexSpace(NL), tL)
    sp = (lambda u, l: (u, l)) if spin else (lambda u, l: None)
    R = tt.Tensor(c, [tv, tv, to, to], spin=sp([0, 1], [2, 3]))
    T = tt.Tensor(c, [tv, tv, to, to], spin=sp([0, 1], [2, 3]))
    X = tt.Tensor(c, [tv, tv, tl], spin=sp([0], [1]))
    lo = L.IndexSpace(O_, [(0, O_ // 2, 1), (O_ // 2, O_, -1)] if spin else [])
    lv = L.IndexSpace(V_, [(0, V_ // 2, 1), (V_ // 2, V_, -1)] if spin else [])
    oo, ov, ol = L.tile_fixed(lo, tO), L.tile_fixed(lv, tV), L.tile_fixed(L.IndexSpace(NL), tL)
    mk = (lambda d, u, l: L.tensor_spin(d, u, l)) if spin else (lambda d, u, l: L.tensor_dense_map(d))
    oR, oT, oX = mk([ov, ov, oo, oo], [0, 1], [2, 3]), mk([ov, ov, oo, oo], [0, 1], [2, 3]), mk([ov, ov, ol], [0], [1])
    return (R, T, X), (oR, oT, oX)


@pytest.mark.parametrize("spin", [False, True])
def test_oracle_cholesky_ladder_cost_closed_forms(spin):
    """The oracle's executed-cost model of the implicit ladder (Eq. cc12) summed over blocks equals the
    closed forms: GEMMs 2 nnz(R) n_W (n_W = v^2 dense, (v/2)^2 with alpha/beta maps: W's (c,d) must
    match the spins of (a,b)), W formation 2 N_L v^2 n_W (every (a,b) row of R is non-zero)."""
    O_, V_, NL = 8, 16, 12
    _, (oR, oT, oX) = _chol_problem(tt, tt.Context(device=-1), O_, V_, 2, 4, NL, 6, spin)
    cb, cost = L.cholesky_ladder_cost(oR, "abij", oX, "abcd", oT, "cdij")
    nnzR = sum(oR.block_volume(b) for b in range(oR.nblocks()) if oR.nz[b])
    nW = (V_ // 2) ** 2 if spin else V_ ** 2
    assert nnzR == (6 * V_ * V_ * O_ * O_ // 16 if spin else V_ * V_ * O_ * O_)
    assert sum(cost) == 2 * nnzR * nW + 2 * NL * V_ * V_ * nW


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("spin", [False, True])
def test_partition_split_cholesky_matches_oracle(nranks, spin):
    """tt_partition_split_cholesky == oracle partition_split on oracle.layout.cholesky_ladder_cost."""
    c = tt.Context(device=-1, nranks=nranks)
    (R, T, X), (oR, oT, oX) = _chol_problem(tt, c, 10, 14, 3, 4, 20, 7, spin)
    cb, cost = L.cholesky_ladder_cost(oR, "abij", oX, "abcd", oT, "cdij")
    exp = L.partition_split(oR, cost, cb, [0, 1], nranks)
    tt.partition_split_cholesky(c, R, "abij", X, "abcd", T, "cdij", group_dims=(0, 1))
    got = {}
    for x in cb:
        if R.owner[x] == tt.TT_SPLIT:
            got[x] = [(lo, hi, o) for (bb, lo, hi, o) in R.parts if bb == x]
        else:
            got[x] = [(0, oR.block_extents(x)[0], int(R.owner[x]))]
    assert got == exp
    with pytest.raises(tt.TTError) as e:   # not the ladder form
        tt.partition_split_cholesky(c, R, "abij", X, "cdab", T, "cdij")
    assert e.value.name == "TT_E_UNSUPPORTED"
