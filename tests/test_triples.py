"""perturbative triples (T), PAPER Eqs. cc13, cc14, tensort, abt, tensort2 (P343-413).

CPU: the oracle (oracle/triples.py) pinned against the DEFINITION <Phi_ijk^abc|V_N X|Phi> evaluated by
second quantization on a tiny Fock space (independent of the printed 18-term expansion; it also fixes
reading R27, the sign of the sixth term), sign / scaling / zero laws of Eq. cc14, and the by-triple
matmul form against the element loops.  GPU: tt_triples_energy against the oracle (normwise on E).
"""
import itertools

import numpy as np
import pytest

from oracle import triples as TR


# ------------------------------------------------------------------------ second quantization (tests only)

def _op(kind, p, det):
    """a_p^+ (kind 'c') or a_p ('a') on a determinant bit string; sign (-1)^(occupied below p)."""
    occ = (det >> p) & 1
    if (kind == "c" and occ) or (kind == "a" and not occ):
        return None, 0
    sign = -1 if bin(det & ((1 << p) - 1)).count("1") % 2 else 1
    return det ^ (1 << p), sign


def _apply(ops, state, coef=1.0, out=None):
    """sum coef * (op_1 op_2 ... op_n) |state>, the rightmost operator acting first."""
    out = {} if out is None else out
    for det, c in state.items():
        d, s = det, c * coef
        for kind, p in reversed(ops):
            d, sg = _op(kind, p, d)
            if d is None:
                break
            s *= sg
        if d is not None:
            out[d] = out.get(d, 0.0) + s
    return out


def _antisym_inputs(nO, nV, seed):
    rng = np.random.default_rng(seed)
    n = nO + nV
    g = rng.uniform(-1, 1, (n, n, n, n))
    g = g + g.transpose(2, 3, 0, 1)                      # real integrals: v^{pq}_{rs} = v^{rs}_{pq}
    v = g - g.transpose(1, 0, 2, 3)
    v = v - v.transpose(0, 1, 3, 2)                      # antisymmetrized <pq||rs>
    t = rng.uniform(-1, 1, (nV, nV, nO, nO))
    t = t - t.transpose(1, 0, 2, 3)
    t = t - t.transpose(0, 1, 3, 2)                      # t^{ij}_{ab} = T2[a,b,i,j], antisymmetric
    t1 = rng.uniform(-1, 1, (nV, nO))
    return v, t, t1


def _slices(v, nO):
    o, w = slice(0, nO), slice(nO, None)
    return v[o, o, o, w], v[w, o, w, w], v[o, o, w, w]   # Vooov(i,j,m,a), Vvovv(e,i,a,b), Voovv(i,j,a,b)


def test_w_and_v1_equal_the_second_quantized_definition():
    """<Phi_ijk^abc| V_N T2 |Phi> and <Phi_ijk^abc| V_N T1 |Phi> with V = 1/4 sum v^{pq}_{rs} a+_p a+_q a_s a_r,
    V_N = V - sum_pq (sum_i v^{pi}_{qi}) a+_p a_q - const (normal order w.r.t. Phi), T2 = 1/4 sum
    t^{ij}_{ab} a+_a a+_b a_j a_i, T1 = sum t^i_a a+_a a_i, |Phi_ijk^abc> = a+_a a+_b a+_c a_k a_j a_i |Phi>
    (P365-369).  Matches Eq. tensort with reading R27 and Eq. tensort2 as printed; the printed sixth
    term ("+") does not."""
    nO, nV = 3, 4
    n = nO + nV
    v, t, t1 = _antisym_inputs(nO, nV, 5)
    phi = {sum(1 << i for i in range(nO)): 1.0}
    vir = range(nO, n)
    T2phi, T1phi = {}, {}
    for i, j in itertools.product(range(nO), repeat=2):
        for a, b in itertools.product(vir, repeat=2):
            _apply([("c", a), ("c", b), ("a", j), ("a", i)], phi, 0.25 * t[a - nO, b - nO, i, j], T2phi)
    for i in range(nO):
        for a in vir:
            _apply([("c", a), ("a", i)], phi, t1[a - nO, i], T1phi)
    gm = np.einsum("piqi->pq", v[:, :nO, :, :nO])
    res2, res1 = {}, {}
    for p, q, r, s in itertools.product(range(n), repeat=4):
        if v[p, q, r, s] != 0.0:
            _apply([("c", p), ("c", q), ("a", s), ("a", r)], T2phi, 0.25 * v[p, q, r, s], res2)
            _apply([("c", p), ("c", q), ("a", s), ("a", r)], T1phi, 0.25 * v[p, q, r, s], res1)
    for p, q in itertools.product(range(n), repeat=2):
        _apply([("c", p), ("a", q)], T2phi, -gm[p, q], res2)
        _apply([("c", p), ("a", q)], T1phi, -gm[p, q], res1)
    Vooov, Vvovv, Voovv = _slices(v, nO)
    checked = 0
    for i, j, k in itertools.combinations(range(nO), 3):
        for a, b, c in itertools.combinations(range(nV), 3):
            ket = _apply([("c", a + nO), ("c", b + nO), ("c", c + nO), ("a", k), ("a", j), ("a", i)], phi)
            w_def = sum(res2.get(d, 0.0) * x for d, x in ket.items())
            v1_def = sum(res1.get(d, 0.0) * x for d, x in ket.items())
            A, B = TR.w_terms(Vooov, Vvovv, t, i, j, k, a, b, c)
            assert abs(A + B - w_def) <= 1e-13 * max(1.0, abs(w_def))
            assert abs(TR.v1_term(Voovv, t1, i, j, k, a, b, c) - v1_def) <= 1e-13 * max(1.0, abs(v1_def))
            # the sixth term as printed ("+") would add 2 * v^{ik}_{mc} t^{mj}_{ab}
            printed = A + B + 2 * float(Vooov[i, k, :, c] @ t[a, b, :, j])
            assert abs(printed - w_def) > 1e-6
            checked += 1
    assert checked == 4


def _random_inputs(nO, nV, seed, antisym=False):
    rng = np.random.default_rng(seed)
    if antisym:
        v, T2, T1 = _antisym_inputs(nO, nV, seed)
        Vooov, Vvovv, Voovv = _slices(v, nO)
    else:
        T1 = rng.uniform(-1, 1, (nV, nO))
        T2 = rng.uniform(-1, 1, (nV, nV, nO, nO))
        Vooov = rng.uniform(-1, 1, (nO, nO, nO, nV))
        Vvovv = rng.uniform(-1, 1, (nV, nO, nV, nV))
        Voovv = rng.uniform(-1, 1, (nO, nO, nV, nV))
    eo = rng.uniform(-2, -1, nO)      # S641 orbital-energy ranges: D < 0
    ev = rng.uniform(1, 2, nV)
    return T1, np.ascontiguousarray(T2), np.ascontiguousarray(Vooov), np.ascontiguousarray(Vvovv), \
        np.ascontiguousarray(Voovv), eo, ev


@pytest.mark.parametrize("nO,nV", [(4, 6), (5, 7), (3, 9)])
def test_energy_by_triple_equals_element_loops(nO, nV):
    args = _random_inputs(nO, nV, nO * 10 + nV)
    E1, n1 = TR.energy(*args)
    E2, n2 = TR.energy_by_triple(*args)
    assert n1 == n2 == (nO * (nO - 1) * (nO - 2) // 6) * (nV * (nV - 1) * (nV - 2) // 6)
    assert abs(E1 - E2) <= 1e-13 * abs(E1)


def test_energy_laws():
    """Eq. cc14: no T2 => W = 0 => E = 0; no T1 => E = sum W^2 / D < 0 (D < 0) and E(lambda T2) = lambda^2 E;
    E is affine in T1 (the second term is linear in T1)."""
    T1, T2, Vooov, Vvovv, Voovv, eo, ev = _random_inputs(4, 6, 1, antisym=True)
    E0, _ = TR.energy(T1, 0 * T2, Vooov, Vvovv, Voovv, eo, ev)
    assert E0 == 0.0
    z = 0 * T1
    E1, _ = TR.energy(z, T2, Vooov, Vvovv, Voovv, eo, ev)
    E3, _ = TR.energy(z, 3 * T2, Vooov, Vvovv, Voovv, eo, ev)
    assert E1 < 0 and abs(E3 - 9 * E1) <= 1e-13 * abs(E3)
    Ea, _ = TR.energy(T1, T2, Vooov, Vvovv, Voovv, eo, ev)
    Eb, _ = TR.energy(2 * T1, T2, Vooov, Vvovv, Voovv, eo, ev)
    assert abs((Eb - E1) - 2 * (Ea - E1)) <= 1e-12 * abs(Eb)


# ------------------------------------------------------------------------------------------ product side

def _spaces(tt, nO, nV, tO, tV, spin):
    if spin:
        O = tt.IndexSpace(nO, [(0, nO // 2), (nO // 2, nO)], [1, -1])
        V = tt.IndexSpace(nV, [(0, nV // 2), (nV // 2, nV)], [1, -1])
    else:
        O, V = tt.IndexSpace(nO), tt.IndexSpace(nV)
    return O, V, tt.TiledIndexSpace(O, tO), tt.TiledIndexSpace(V, tV)


def _oracle_dims(nO, nV, tO, tV, spin):
    from oracle import layout as L
    if spin:
        O = L.IndexSpace(nO, [(0, nO // 2, 1), (nO // 2, nO, -1)])
        V = L.IndexSpace(nV, [(0, nV // 2, 1), (nV // 2, nV, -1)])
    else:
        O, V = L.IndexSpace(nO), L.IndexSpace(nV)
    return L.tile_fixed(O, tO), L.tile_fixed(V, tV)


# (name, dims as 'o'/'v', spin (upper dims, lower dims), generator tag)
TRIPLES_INPUTS = [("T1", "vo", ([0], [1]), 11), ("T2", "vvoo", ([0, 1], [2, 3]), 12),
                  ("Vooov", "ooov", ([0, 1], [2, 3]), 13), ("Vvovv", "vovv", ([0, 1], [2, 3]), 14),
                  ("Voovv", "oovv", ([0, 1], [2, 3]), 15)]


def _expected_units(nO, nV, spin, box=16):
    """Units of the fused kernel: (occupied triple i<j<k) x (16-wide virtual box triple with at least one
    a<b<c), spin sums equal (alpha = first half, R6)."""
    def sp(n, x):
        return (1 if x < n // 2 else -1) if spin else 0
    ranges = [(0, nV // 2), (nV // 2, nV)] if spin else [(0, nV)]
    boxes = [(x, min(box, e - x), sp(nV, x)) for b, e in ranges for x in range(b, e, box)]
    count = 0
    occ = [sum(sp(nO, x) for x in t) for t in itertools.combinations(range(nO), 3)]
    for A, B, C in itertools.combinations_with_replacement(boxes, 3):
        n = sum(1 for a in range(A[0], A[0] + A[1]) for b in range(B[0], B[0] + B[1]) for c in range(C[0], C[0] + C[1])
                if a < b < c)
        if n:
            count += sum(1 for o in occ if o == A[2] + B[2] + C[2])
    return count


@pytest.mark.parametrize("nO,nV,tO,tV,spin", [(7, 10, 3, 4, False), (8, 12, 2, 3, True), (6, 40, 1, 10, False),
                                                (8, 68, 2, 17, True)])
def test_triples_plan_host(nO, nV, tO, tV, spin):
    import paper_2201_01257_b200 as tt
    ctx = tt.Context(device=-1)
    O, V, to, tv = _spaces(tt, nO, nV, tO, tV, spin)
    dims = {"o": to, "v": tv}
    T = {n: tt.Tensor(ctx, [dims[c] for c in d], spin=sp if spin else None) for n, d, sp, _ in TRIPLES_INPUTS}
    _, info = tt.triples_energy(ctx, T["T1"], T["T2"], T["Vooov"], T["Vvovv"], T["Voovv"])
    assert info["w_blocks_total"] == info["w_blocks"] == _expected_units(nO, nV, spin)
    if not spin:   # every restricted element once: 18 (n_o + n_v) FLOPs each
        n = (nO * (nO - 1) * (nO - 2) // 6) * (nV * (nV - 1) * (nV - 2) // 6)
        assert info["flops_alg"] == pytest.approx(18.0 * (nO + nV) * n, rel=1e-12)
    # a dimension on another tiling object is refused
    other = tt.TiledIndexSpace(V, tV)
    bad = tt.Tensor(ctx, [to, to, tv, other])
    with pytest.raises(tt.TTError) as e:
        tt.triples_energy(ctx, T["T1"], T["T2"], T["Vooov"], T["Vvovv"], bad)
    assert e.value.name == "TT_E_TILING"


def _gpu_case(nO, nV, tO, tV, spin, seed, ws_factor):
    import torch
    import paper_2201_01257_b200 as tt
    import synthetic as S
    from oracle import layout as L
    from oracle import ops as O_
    ctx = tt.Context(device=0, stream=torch.cuda.current_stream().cuda_stream)
    _, _, to, tv = _spaces(tt, nO, nV, tO, tV, spin)
    oO, oV = _oracle_dims(nO, nV, tO, tV, spin)
    dims, odims = {"o": to, "v": tv}, {"o": oO, "v": oV}
    T, dense, keep = {}, {}, []
    for n, d, sp, tag in TRIPLES_INPUTS:
        T[n] = tt.Tensor(ctx, [dims[c] for c in d], spin=sp if spin else None)
        ot = L.tensor_spin([odims[c] for c in d], *sp) if spin else L.tensor_dense_map([odims[c] for c in d])
        dense[n] = O_.dense_masked(ot, S.dense(ot.shape, seed, tag))
        buf = torch.from_numpy(O_.pack(ot, dense[n])).cuda()
        T[n].bind(buf)
        keep.append(buf)
    rng = np.random.default_rng(seed)
    eo, ev = rng.uniform(-2, -1, nO), rng.uniform(1, 2, nV)
    deo, dev = torch.from_numpy(eo).cuda(), torch.from_numpy(ev).cuda()
    args = (T["T1"], T["T2"], T["Vooov"], T["Vvovv"], T["Voovv"])
    _, info = tt.triples_energy(ctx, *args)
    ws = torch.empty(int(info["ws_elems"] * ws_factor), dtype=torch.float64, device="cuda")
    E, info = tt.triples_energy(ctx, *args, deo, dev, ws)
    orc = (dense["T1"], dense["T2"], dense["Vooov"], dense["Vvovv"], dense["Voovv"], eo, ev)
    return E, info, orc, ctx


@pytest.mark.gpu
@pytest.mark.parametrize("nO,nV,tO,tV,spin", [(7, 10, 3, 4, False), (8, 12, 2, 3, True), (6, 22, 4, 5, False)])
def test_triples_energy_gpu_parity(nO, nV, tO, tV, spin):
    E, info, orc, _ = _gpu_case(nO, nV, tO, tV, spin, 3, 50.0)
    Eo, n = TR.energy(*orc)
    scale = sum(abs(c[0]) for c in TR.energy_elements(*orc, [(i, j, k, a, b, c)
                for i, j, k in itertools.combinations(range(nO), 3) for a, b, c in itertools.combinations(range(nV), 3)]))
    assert abs(E - Eo) <= 1e-11 * scale, (E, Eo, scale)
    assert info["flops_alg"] <= info["flops_exec"]
    if not spin:
        assert info["flops_alg"] == pytest.approx(18.0 * (nO + nV) * n, rel=1e-12)


@pytest.mark.gpu
def test_triples_deterministic():
    """Fixed partial order and fixed final tree (R12): two calls give the same bits."""
    import torch
    import paper_2201_01257_b200 as tt
    E1, i1, _, ctx = _gpu_case(7, 22, 2, 3, False, 4, 1.0)
    E2, i2, _, _ = _gpu_case(7, 22, 2, 3, False, 4, 1.0)
    assert E1 == E2


@pytest.mark.gpu
def test_triples_energy_gpu_parity_midsize():
    """Several tiles per space with ragged tails (O=16 tiles 5,5,5,1; V=48 tiles 10 x4 + 8; three 16-wide boxes);
    oracle = the by-triple form (pinned to the element loops above)."""
    E, info, orc, _ = _gpu_case(16, 48, 5, 10, False, 7, 1.0)
    Eo, n = TR.energy_by_triple(*orc)
    assert abs(E - Eo) <= 1e-11 * abs(Eo), (E, Eo)
    assert info["flops_alg"] == pytest.approx(18.0 * (16 + 48) * n, rel=1e-12)


@pytest.mark.gpu
def test_triples_energy_gpu_parity_spin_boxes():
    """alpha/beta maps with two 16-wide boxes per spin range (V = 36: 18 per range = 16 + 2), spin-forbidden
    units skipped; oracle = the by-triple form over the dense masked inputs."""
    E, info, orc, _ = _gpu_case(8, 36, 2, 9, True, 9, 1.0)
    Eo, n = TR.energy_by_triple(*orc)
    assert abs(E - Eo) <= 1e-11 * abs(Eo), (E, Eo)


def test_triples_odd_virtual_range_refused():
    import paper_2201_01257_b200 as tt
    ctx = tt.Context(device=-1)
    _, _, to, tv = _spaces(tt, 6, 9, 2, 3, False)
    dims = {"o": to, "v": tv}
    T = {n: tt.Tensor(ctx, [dims[c] for c in d]) for n, d, sp, _ in TRIPLES_INPUTS}
    with pytest.raises(tt.TTError) as e:
        tt.triples_energy(ctx, T["T1"], T["T2"], T["Vooov"], T["Vvovv"], T["Voovv"])
    assert e.value.name == "TT_E_UNSUPPORTED"


@pytest.mark.parametrize("nO,nV,tO,tV,spin,nranks", [(7, 20, 3, 5, False, 3), (8, 40, 2, 10, True, 4),
                                                       (9, 36, 3, 9, False, 2)])
def test_triples_units_partition_over_ranks(nO, nV, tO, tV, spin, nranks):
    """Units split into contiguous ranges of equal modelled cost: the counts sum to the total, the rank
    costs sum to the total cost, and each rank is within one unit's cost of total / nranks."""
    import paper_2201_01257_b200 as tt
    counts, costs, flops = [], [], []
    for r in range(nranks):
        ctx = tt.Context(device=-1, rank=r, nranks=nranks)
        _, _, to, tv = _spaces(tt, nO, nV, tO, tV, spin)
        dims = {"o": to, "v": tv}
        T = {n: tt.Tensor(ctx, [dims[c] for c in d], spin=sp if spin else None) for n, d, sp, _ in TRIPLES_INPUTS}
        for X in T.values():
            X.set_owner(np.full(X.nblocks, tt.TT_REPLICATED, np.int32))
        _, info = tt.triples_energy(ctx, T["T1"], T["T2"], T["Vooov"], T["Vvovv"], T["Voovv"])
        counts.append(info["w_blocks"])
        costs.append(info["cost_rank"])
        flops.append(info["flops_exec"])
        total, ctotal, cmax = info["w_blocks_total"], info["cost_total"], info["cost_max_unit"]
    assert sum(counts) == total == _expected_units(nO, nV, spin)
    assert sum(costs) == pytest.approx(ctotal, rel=1e-12)
    assert max(abs(c - ctotal / nranks) for c in costs) <= cmax
    assert sum(flops) == _expected_exec_flops(nO, nV, spin)


def _expected_exec_flops(nO, nV, spin, box=16):
    """DMMA FLOPs the default kernel issues, counted by brute force: per unit and GEMM g (row role = index
    g of (a,b,c); columns = (p, q) with p the first remaining index and q the other), every 8-row x
    (one p, 8 q) output fragment holding an element a<b<c inside the boxes, times the 8-row stages of its
    m and e segments (spin: only the allowed half of each sum), x 2 x 8 x 8 x 8 per fragment-stage."""
    def sp(n, x):
        return (1 if x < n // 2 else -1) if spin else 0
    ranges = [(0, nV // 2), (nV // 2, nV)] if spin else [(0, nV)]
    boxes = [(x, min(box, e - x), sp(nV, x)) for b, e in ranges for x in range(b, e, box)]
    half_o, half_v = (nO // 2, nV // 2) if spin else (0, 0)

    def seg(n, half, s):           # stages of a sum over n indices restricted to spin s (0 = no spin)
        ln = n if not half else (half if s == 1 else (n - half if s == -1 else 0))
        return -(-ln // 8)
    total = 0
    for bx in itertools.combinations_with_replacement(boxes, 3):
        if not any(a < b < c for a in range(bx[0][0], bx[0][0] + bx[0][1]) for b in range(bx[1][0], bx[1][0] + bx[1][1])
                   for c in range(bx[2][0], bx[2][0] + bx[2][1])):
            continue
        for i, j, k in itertools.combinations(range(nO), 3):
            if spin and sp(nO, i) + sp(nO, j) + sp(nO, k) != bx[0][2] + bx[1][2] + bx[2][2]:
                continue
            for g in range(3):
                roles = [g] + [d for d in range(3) if d != g]      # row, p, q
                nf = 0
                for r0 in (0, 8):
                    for p in range(box):
                        for q0 in (0, 8):
                            cell = {roles[0]: range(r0, min(r0 + 8, bx[roles[0]][1])),
                                    roles[1]: range(p, min(p + 1, bx[roles[1]][1])),
                                    roles[2]: range(q0, min(q0 + 8, bx[roles[2]][1]))}
                            if any(bx[0][0] + x < bx[1][0] + y < bx[2][0] + z
                                   for x in cell[0] for y in cell[1] for z in cell[2]):
                                nf += 1
                # segments: m sums over v^{xy}_{m r} (s_m = s_x + s_y - s_r), e sums over v^{ex}_{pq}
                # (s_e = s_p + s_q - s_x), occupied pairs / singles of the three terms of G
                so = [sp(nO, i), sp(nO, j), sp(nO, k)]
                sr, spp, sq = bx[roles[0]][2], bx[roles[1]][2], bx[roles[2]][2]
                st = sum(seg(nO, half_o, so[x] + so[y] - sr) for x, y in ((0, 1), (0, 2), (1, 2)))
                st += sum(seg(nV, half_v, spp + sq - so[x]) for x in range(3))
                total += nf * st * 2 * 8 * 8 * 8
    return total


@pytest.mark.gpu
@pytest.mark.parametrize("tma,pair,cluster,code", [("0", "0", "0", 0), ("1", "0", "0", 1), ("1", "1", "0", 2),
                                                  ("1", "0", "1", 3)])
def test_triples_all_kernel_variants(tma, pair, cluster, code):
    """cp.async staging (TT_TMA=0), TMA boxes one unit per CTA, the opt-in 16-warp pair kernel
    (TT_TRIPLES_PAIR=1) and the opt-in 2-CTA cluster kernel with TMA multicast of the shared operand
    (TT_TRIPLES_CLUSTER=1) give the oracle's energy -- bitwise the same energy, since every unit's partial is formed in
    the same order; O, V not multiples of the 8-row stage (segment tails are zero fill)."""
    import os
    os.environ["TT_TMA"], os.environ["TT_TRIPLES_PAIR"], os.environ["TT_TRIPLES_CLUSTER"] = tma, pair, cluster
    try:
        E, info, orc, ctx = _gpu_case(13, 38, 4, 7, False, 11, 1.0)
        assert ctx.stats()["producer"] == code
    finally:
        for k in ("TT_TMA", "TT_TRIPLES_PAIR", "TT_TRIPLES_CLUSTER"):
            os.environ.pop(k, None)
    Eo, _ = TR.energy_by_triple(*orc)
    assert abs(E - Eo) <= 1e-11 * abs(Eo), (E, Eo)
    _ENERGIES.setdefault("v", set()).add(E)
    assert len(_ENERGIES["v"]) == 1


_ENERGIES = {}


def test_triples_algorithmic_flops_spin_brute_force():
    """flops_alg = 2 per non-zero product of the 18 terms over the restricted spin-allowed elements: counted
    here element by element from the spin rule of R7 (v^{xy}_{m p} needs s_m = s_x + s_y - s_p, v^{e x}_{p q}
    needs s_e = s_p + s_q - s_x)."""
    import paper_2201_01257_b200 as tt
    nO, nV = 8, 20
    ctx = tt.Context(device=-1)
    _, _, to, tv = _spaces(tt, nO, nV, 2, 5, True)
    dims = {"o": to, "v": tv}
    T = {n: tt.Tensor(ctx, [dims[c] for c in d], spin=sp) for n, d, sp, _ in TRIPLES_INPUTS}
    _, info = tt.triples_energy(ctx, T["T1"], T["T2"], T["Vooov"], T["Vvovv"], T["Voovv"])
    so = [1 if x < nO // 2 else -1 for x in range(nO)]
    sv = [1 if x < nV // 2 else -1 for x in range(nV)]
    nm = {1: sum(1 for x in so if x == 1), -1: sum(1 for x in so if x == -1)}
    ne = {1: sum(1 for x in sv if x == 1), -1: sum(1 for x in sv if x == -1)}
    total = 0
    for i, j, k in itertools.combinations(range(nO), 3):
        for a, b, c in itertools.combinations(range(nV), 3):
            if so[i] + so[j] + so[k] != sv[a] + sv[b] + sv[c]:
                continue
            n = 0
            for x, y in ((i, j), (i, k), (j, k)):          # A terms: v^{xy}_{m p}, p in (a, b, c)
                for p in (a, b, c):
                    n += nm.get(so[x] + so[y] - sv[p], 0)
            for x in (i, j, k):                             # B terms: v^{e x}_{p q}, (p, q) in (ab, ac, bc)
                for p, q in ((a, b), (a, c), (b, c)):
                    n += ne.get(sv[p] + sv[q] - so[x], 0)
            total += 2 * n
    assert info["flops_alg"] == total


def test_triples_argument_errors():
    """Too small a workspace -> TT_E_OOM; missing orbital energies -> TT_E_ARG (checked before any launch)."""
    import paper_2201_01257_b200 as tt
    ctx = tt.Context(device=-1)
    _, _, to, tv = _spaces(tt, 6, 10, 2, 4, False)
    dims = {"o": to, "v": tv}
    T = {n: tt.Tensor(ctx, [dims[c] for c in d]) for n, d, sp, _ in TRIPLES_INPUTS}
    args = (T["T1"], T["T2"], T["Vooov"], T["Vvovv"], T["Voovv"])
    _, info = tt.triples_energy(ctx, *args)
    fake = 1 << 20   # never dereferenced: the calls fail during validation
    with pytest.raises(tt.TTError) as e:
        tt.triples_energy(ctx, *args, fake, fake, fake, ws_elems=info["ws_elems"] - 2)
    assert e.value.name == "TT_E_OOM"
    with pytest.raises(tt.TTError) as e:
        tt.triples_energy(ctx, *args, None, fake, fake, ws_elems=info["ws_elems"])
    assert e.value.name == "TT_E_ARG"


def test_triples_rejects_maps_outside_the_spin_rule():
    """The kernel prunes units and m / e ranges by the index spins (R28): on alpha/beta spaces an input
    with a dense block map (blocks outside the R7 spin map) must be refused, not mis-summed;
    the spin maps themselves pass, and dense maps on spaces without spin pass."""
    import paper_2201_01257_b200 as tt
    ctx = tt.Context(device=-1)
    _, _, to, tv = _spaces(tt, 6, 12, 3, 3, True)
    dims = {"o": to, "v": tv}
    spin = {n: tt.Tensor(ctx, [dims[c] for c in d], spin=sp) for n, d, sp, _ in TRIPLES_INPUTS}
    args = [spin[n] for n in ("T1", "T2", "Vooov", "Vvovv", "Voovv")]
    tt.triples_energy(ctx, *args)                       # query mode: spin maps accepted
    for k, (n, d, sp, _) in enumerate(TRIPLES_INPUTS):
        bad = list(args)
        bad[k] = tt.Tensor(ctx, [dims[c] for c in d])   # dense map on spin spaces
        with pytest.raises(tt.TTError) as e:
            tt.triples_energy(ctx, *bad)
        assert e.value.name == "TT_E_UNSUPPORTED" and n in e.value.args[0]
    _, _, to2, tv2 = _spaces(tt, 6, 12, 3, 3, False)
    d2 = {"o": to2, "v": tv2}
    dense = [tt.Tensor(ctx, [d2[c] for c in d]) for n, d, sp, _ in TRIPLES_INPUTS]
    tt.triples_energy(ctx, *dense)


@pytest.mark.gpu
@pytest.mark.parametrize("p", [2, 3])
def test_triples_owner_distributed_inputs_simulated_ranks(p):
    """With several ranks the inputs may be owner-distributed (round robin here, non-held blocks NaN):
    each rank gathers what it does not hold before re-tiling, the units split by cost, and every rank
    returns the same energy as one rank, within 1e-11 of the oracle (simulated ranks on one GPU)."""
    import torch
    import paper_2201_01257_b200 as tt
    import synthetic as S
    from oracle import layout as L
    from oracle import ops as O_
    from tests.simranks import run_ranks
    nO, nV, tO, tV, spin, seed = 8, 20, 2, 5, True, 4
    oO, oV = _oracle_dims(nO, nV, tO, tV, spin)
    odims = {"o": oO, "v": oV}
    dense, packed = {}, {}
    for n, d, sp, tag in TRIPLES_INPUTS:
        ot = L.tensor_spin([odims[c] for c in d], *sp)
        dense[n] = O_.dense_masked(ot, S.dense(ot.shape, seed, tag))
        packed[n] = O_.pack(ot, dense[n])
    rng = np.random.default_rng(seed)
    eo, ev = rng.uniform(-2, -1, nO), rng.uniform(1, 2, nV)

    def body(rank, ctx):
        _, _, to, tv = _spaces(tt, nO, nV, tO, tV, spin)
        dims = {"o": to, "v": tv}
        T, keep = {}, []
        for n, d, sp, _ in TRIPLES_INPUTS:
            X = tt.Tensor(ctx, [dims[c] for c in d], spin=sp)
            X.set_owner(np.where(X.nz > 0, np.arange(X.nblocks) % ctx.nranks, -1).astype(np.int32))
            host = packed[n].copy()
            for blk in range(X.nblocks):   # only the owned blocks hold data
                if X.nz[blk] and X.owner[blk] != rank:
                    o = int(X.blk_off[blk])
                    ext = [int(dd.offsets[t + 1] - dd.offsets[t]) for dd, t in zip(X.dims, np.unravel_index(blk, X.grid))]
                    host[o:o + int(np.prod(ext))] = np.nan
            buf = torch.from_numpy(host).cuda()
            X.bind(buf)
            T[n] = X
            keep.append(buf)
        args = (T["T1"], T["T2"], T["Vooov"], T["Vvovv"], T["Voovv"])
        _, info = tt.triples_energy(ctx, *args)
        ws = torch.empty(int(info["ws_elems"] * 1.5), dtype=torch.float64, device="cuda")
        E, _ = tt.triples_energy(ctx, *args, torch.from_numpy(eo).cuda(), torch.from_numpy(ev).cuda(), ws)
        ctx.sync()
        return E

    E1 = run_ranks(tt, torch, 1, body)[0]
    Ep = run_ranks(tt, torch, p, body)
    assert all(np.isfinite(e) for e in Ep) and len(set(Ep)) == 1, Ep
    assert abs(Ep[0] - E1) <= 1e-13 * abs(E1)
    orc = (dense["T1"], dense["T2"], dense["Vooov"], dense["Vvovv"], dense["Voovv"], eo, ev)
    Eo, _ = TR.energy(*orc)
    scale = sum(abs(c[0]) for c in TR.energy_elements(*orc, [(i, j, k, a, b, c)
                for i, j, k in itertools.combinations(range(nO), 3) for a, b, c in itertools.combinations(range(nV), 3)]))
    assert abs(E1 - Eo) <= 1e-11 * scale, (E1, Eo, scale)
