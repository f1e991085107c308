"""GPU parity: libtt (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bar (BASELINE north_star, reading R13): normwise max|gpu - oracle| / max|oracle| <= 1e-11 per output
tensor for uniform inputs; bit-exact for integer-valued inputs, tile maps, task lists and the
synthetic fill.  Sizes span several CTA tiles with ragged tails; edge cases: ragged tiles, permuted
labels, beta = 0 with NaN in C, C blocks without tasks, every kernel tile variant, determinism."""
import os

import numpy as np
import pytest

import synthetic as S
from oracle import layout as L
from oracle import ops as O
from tests.cases import Problem, SpaceSpec, TensorSpec, ccsd_problem, oracle_objects, product_objects

pytestmark = pytest.mark.gpu

TOL = 1e-11


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2201_01257_b200 as tt
    torch.cuda.init()
    return tt, torch


def new_ctx(tt, torch, variant=None):
    if variant is None:
        os.environ.pop("TT_FORCE_VARIANT", None)
    else:
        os.environ["TT_FORCE_VARIANT"] = str(variant)
    return tt.Context(device=0, stream=torch.cuda.current_stream().cuda_stream)


def bind_host(torch, T, packed):
    dev = torch.from_numpy(np.ascontiguousarray(packed)).cuda()
    T.bind(dev)
    return dev


def normwise(x, ref):
    return float(np.abs(x - ref).max() / max(np.abs(ref).max(), 1e-300)) if ref.size else 0.0


def run_contract(tt, torch, ctx, pb, op, alpha=1.0, beta=1.0, kind=S.KIND_UNIFORM, seed=1, nan_c=False):
    C, cl, a, al, b, bl = op
    orc = oracle_objects(pb)
    P = product_objects(tt, ctx, pb)
    dense = {}
    bufs = []
    for name, tag in ((C, 3), (a, 1), (b, 2)):
        D = O.dense_masked(orc[name], S.dense(orc[name].shape, seed, tag, kind))
        if name == C and nan_c:
            D = np.where(O.nz_mask(orc[name]).astype(bool), np.nan, 0.0)
        dense[name] = D
        bufs.append(bind_host(torch, P[name], O.pack(orc[name], D)))
    tt.contract(ctx, P[C], cl, beta, alpha, P[a], al, P[b], bl)
    got = P[C].download()
    ctx.sync()
    ref = O.contract(dense[C], cl, dense[a], al, dense[b], bl, alpha, beta, cmask=O.nz_mask(orc[C]))
    return got, O.pack(orc[C], ref), P, orc


PROBLEMS = {
    "cfg1_ring_dense": (ccsd_problem(4, 8, 4, 4, False, terms=("ring",)), 0),
    "spin_small_ladder": (ccsd_problem(8, 12, 2, 3, True), 0),
    "spin_small_ring": (ccsd_problem(8, 12, 2, 3, True), 1),
    "spin_small_hh": (ccsd_problem(8, 12, 2, 3, True), 2),
    "ragged_dense_ring": (ccsd_problem(7, 13, 3, 5, False), 1),
    "ragged_dense_ladder": (ccsd_problem(7, 13, 3, 5, False), 0),
    "multi_tile_spin_ladder": (ccsd_problem(24, 80, 12, 20, True, terms=("ladder",)), 0),
    "multi_tile_spin_ring": (ccsd_problem(24, 80, 12, 20, True, terms=("ring",)), 0),
}


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_contract_parity(env, name):
    tt, torch = env
    pb, k = PROBLEMS[name]
    ctx = new_ctx(tt, torch)
    got, ref, _, _ = run_contract(tt, torch, ctx, pb, pb.ops[k], alpha=0.75, beta=1.0)
    assert normwise(got, ref) <= TOL, normwise(got, ref)


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 5])
def test_every_tile_variant(env, variant):
    tt, torch = env
    pb = ccsd_problem(24, 80, 12, 20, True, terms=("ladder", "ring"))
    ctx = new_ctx(tt, torch, variant)
    for op in pb.ops:
        got, ref, _, _ = run_contract(tt, torch, ctx, pb, op, alpha=1.5, beta=-0.5)
        assert normwise(got, ref) <= TOL
        assert ctx.stats()["kernel_variant"] == variant
    os.environ.pop("TT_FORCE_VARIANT", None)


def test_integer_inputs_bit_exact(env):
    tt, torch = env
    pb = ccsd_problem(12, 30, 6, 10, True)
    ctx = new_ctx(tt, torch)
    for op in pb.ops:
        got, ref, _, _ = run_contract(tt, torch, ctx, pb, op, alpha=2.0, beta=1.0, kind=S.KIND_INTEGER)
        assert np.array_equal(got, ref)


def test_beta_zero_never_reads_c(env):
    tt, torch = env
    pb = ccsd_problem(8, 12, 2, 3, True)
    ctx = new_ctx(tt, torch)
    for op in pb.ops:
        got, ref, _, _ = run_contract(tt, torch, ctx, pb, op, alpha=0.5, beta=0.0, nan_c=True)
        assert np.isfinite(got).all()
        assert normwise(got, np.nan_to_num(ref)) <= TOL


@pytest.mark.parametrize("variant", [None, 1, 3, 4, 5])
@pytest.mark.parametrize("even", [False, True])
def test_permuted_labels(env, variant, even):
    """Operands whose innermost labels are free/contracted in every combination (all four kernel
    orientations; with even tiles also the 16-byte copy paths), output permuted relative to both."""
    tt, torch = env
    if even:
        spaces = {"X": SpaceSpec(12, tile=4), "Y": SpaceSpec(10, tile=6), "Z": SpaceSpec(14, tile=8)}
    else:
        spaces = {"X": SpaceSpec(11, tile=4), "Y": SpaceSpec(9, tile=5), "Z": SpaceSpec(10, tile=3)}
    ls = {"a": "X", "b": "Y", "c": "Z", "i": "Y", "j": "X", "k": "Z"}
    ctx = new_ctx(tt, torch, variant)
    for cl, al, bl in [("jbia", "kcai", "bjck"), ("abij", "iack", "kcjb"), ("ijab", "akci", "jbkc"),
                       ("bjai", "ciak", "cbkj")]:
        tens = {"C": TensorSpec(cl), "A": TensorSpec(al), "B": TensorSpec(bl)}
        pb = Problem(spaces, ls, tens, [("C", cl, "A", al, "B", bl)])
        got, ref, _, _ = run_contract(tt, torch, ctx, pb, pb.ops[0], alpha=1.0, beta=0.5)
        assert normwise(got, ref) <= TOL, (cl, al, bl)
    os.environ.pop("TT_FORCE_VARIANT", None)


def test_c_blocks_without_tasks(env):
    """Non-zero C blocks with no non-zero (A,B) pair get C = beta*C (A8 / S509)."""
    tt, torch = env
    spaces = {"X": SpaceSpec(12, tile=4)}
    ls = {x: "X" for x in "ikl"}
    nzA = [1, 0, 0, 0, 1, 0, 1, 0, 0]     # A blocks (i,k): row 2 has A(2,0) only
    nzB = [0, 1, 1, 0, 1, 0, 0, 0, 1]     # B(0,*) zero except cols 1,2 ...
    pb = Problem(spaces, ls, {"C": TensorSpec("il"), "A": TensorSpec("ik", ("nz", nzA)), "B": TensorSpec("kl", ("nz", nzB))},
                 [("C", "il", "A", "ik", "B", "kl")])
    ctx = new_ctx(tt, torch)
    got, ref, P, _ = run_contract(tt, torch, ctx, pb, pb.ops[0], alpha=1.0, beta=-2.0)
    assert normwise(got, ref) <= TOL


def test_determinism(env):
    tt, torch = env
    pb = ccsd_problem(24, 80, 12, 20, True, terms=("ring",))
    ctx = new_ctx(tt, torch)
    g1, _, _, _ = run_contract(tt, torch, ctx, pb, pb.ops[0], seed=5)
    g2, _, _, _ = run_contract(tt, torch, ctx, pb, pb.ops[0], seed=5)
    assert np.array_equal(g1, g2)


@pytest.mark.parametrize("splitk", [2, 3, 7])
@pytest.mark.parametrize("variant", [None, 1, 3, 5])
def test_split_k_forced(env, splitk, variant):
    """Task lists cut into up to `splitk` chunks (partial sums reduced in chunk order): parity on
    ladder / ring / hole-hole terms, beta = 0 with NaN in C, permuted labels; deterministic."""
    tt, torch = env
    os.environ["TT_SPLITK"] = str(splitk)
    try:
        pb = ccsd_problem(12, 30, 3, 5, True)
        ctx = new_ctx(tt, torch, variant)
        for op in pb.ops:
            got, ref, _, _ = run_contract(tt, torch, ctx, pb, op, alpha=1.25, beta=-0.5)
            assert normwise(got, ref) <= TOL
            got2, ref2, _, _ = run_contract(tt, torch, ctx, pb, op, alpha=0.5, beta=0.0, nan_c=True)
            assert np.isfinite(got2).all() and normwise(got2, np.nan_to_num(ref2)) <= TOL
            got3, _, _, _ = run_contract(tt, torch, ctx, pb, op, alpha=1.25, beta=-0.5)
            assert np.array_equal(got, got3)
        spaces = {"X": SpaceSpec(11, tile=4), "Y": SpaceSpec(9, tile=5), "Z": SpaceSpec(10, tile=3)}
        ls = {"a": "X", "b": "Y", "c": "Z", "i": "Y", "j": "X", "k": "Z"}
        for cl, al, bl in [("jbia", "kcai", "bjck"), ("ijab", "akci", "jbkc")]:
            tens = {"C": TensorSpec(cl), "A": TensorSpec(al), "B": TensorSpec(bl)}
            q = Problem(spaces, ls, tens, [("C", cl, "A", al, "B", bl)])
            got, ref, _, _ = run_contract(tt, torch, ctx, q, q.ops[0], alpha=1.0, beta=0.5)
            assert normwise(got, ref) <= TOL, (cl, al, bl)
    finally:
        os.environ.pop("TT_SPLITK", None)
        os.environ.pop("TT_FORCE_VARIANT", None)


def test_split_k_small_output_large_k(env):
    """Hole-hole-shaped C(m,i) += A(e,f,m,n) B(e,f,i,n): few output tiles, long task lists -- the
    planner splits K on its own (one launch of the reduce kernel), parity and bitwise equality with
    the row-split (parts) version of the same C (chunking independent of the part rows)."""
    tt, torch = env
    spaces = {"O": SpaceSpec(12, tile=6), "V": SpaceSpec(120, tile=10)}
    ls = {"m": "O", "i": "O", "n": "O", "e": "V", "f": "V"}
    tens = {"C": TensorSpec("mi"), "A": TensorSpec("efmn"), "B": TensorSpec("efin")}
    pb = Problem(spaces, ls, tens, [("C", "mi", "A", "efmn", "B", "efin")])
    ctx = new_ctx(tt, torch)
    got, ref, P, orc = run_contract(tt, torch, ctx, pb, pb.ops[0], alpha=0.5, beta=1.0, seed=6)
    assert normwise(got, ref) <= TOL
    assert ctx.stats()["work_items"] > 4          # 4 C blocks, chunked
    ctx2 = new_ctx(tt, torch)
    orc2 = oracle_objects(pb)
    P2 = product_objects(tt, ctx2, pb)
    _split_all(P2["C"], 2)
    bufs = []
    for name, tag in (("C", 3), ("A", 1), ("B", 2)):
        bufs.append(bind_host(torch, P2[name], O.pack(orc2[name], O.dense_masked(orc2[name], S.dense(orc2[name].shape, 6, tag)))))
    tt.contract(ctx2, P2["C"], "mi", 1.0, 0.5, P2["A"], "efmn", P2["B"], "efin")
    g2 = P2["C"].download()
    ctx2.sync()
    assert np.array_equal(got, g2)


@pytest.mark.parametrize("pi", [0, 1])
def test_device_task_list_bit_exact(env, pi):
    tt, torch = env
    pb = [ccsd_problem(8, 12, 2, 3, True), ccsd_problem(60, 400, 30, 40, True)][pi]
    ctx = new_ctx(tt, torch)
    orc = oracle_objects(pb)
    P = product_objects(tt, ctx, pb)
    for (c, cl, a, al, b, bl) in pb.ops:
        ocb, optr, oab, obb, ocost = L.task_list(orc[c], cl, orc[a], al, orc[b], bl)
        tl = tt.task_list(ctx, P[c], cl, P[a], al, P[b], bl, device=True)
        assert list(tl["cblk"]) == ocb and list(tl["ptr"]) == optr
        assert list(tl["a_blk"]) == oab and list(tl["b_blk"]) == obb


@pytest.mark.parametrize("kind", [S.KIND_UNIFORM, S.KIND_INTEGER])
def test_fill_synthetic_bit_exact(env, kind):
    tt, torch = env
    pb = ccsd_problem(10, 14, 3, 4, True, terms=("ring",))
    ctx = new_ctx(tt, torch)
    orc = oracle_objects(pb)
    P = product_objects(tt, ctx, pb)
    for name in ("Ta", "Wr", "R"):
        buf = torch.zeros(P[name].packed_elems, dtype=torch.float64, device="cuda")
        P[name].bind(buf)
        tt.fill_synthetic(ctx, P[name], 7, 4, kind)
        got = P[name].download()
        ctx.sync()
        ref = O.pack(orc[name], S.dense(orc[name].shape, 7, 4, kind))
        assert np.array_equal(got, ref)


def test_set_add_scalar(env):
    tt, torch = env
    pb = ccsd_problem(8, 12, 2, 3, True)
    pb.tensors["Rt"] = TensorSpec("ijab", ("spin", [0, 1], [2, 3]))
    ctx = new_ctx(tt, torch)
    orc = oracle_objects(pb)
    P = product_objects(tt, ctx, pb)
    bufs = {}
    dense = {}
    for name, tag in (("R", 3), ("Rt", 1), ("Ta", 2)):
        dense[name] = O.dense_masked(orc[name], S.dense(orc[name].shape, 3, tag))
        bufs[name] = bind_host(torch, P[name], O.pack(orc[name], dense[name]))
    # add with permutation: R(abij) = -0.5*R + 2*Rt(ijab)
    tt.add(ctx, P["R"], "abij", -0.5, 2.0, P["Rt"], "ijab")
    got = P["R"].download()
    ctx.sync()
    ref = O.add(dense["R"], "abij", dense["Rt"], "ijab", 2.0, -0.5, cmask=O.nz_mask(orc["R"]))
    assert normwise(got, O.pack(orc["R"], ref)) <= 1e-15
    # scalar: s = 0.25 * sum Ta(acik) R(acik)  (relabelled R)
    R2 = ref
    s = tt.contract_scalar(ctx, 0.25, P["Ta"], "acik", P["R"], "acik")
    so = O.scalar(dense["Ta"], "acik", R2, "acik", 0.25)
    assert abs(s - so) <= 1e-13 * max(abs(so), 1.0)
    # set
    tt.set_(ctx, P["R"], 3.25)
    got = P["R"].download()
    ctx.sync()
    assert np.array_equal(got, O.pack(orc["R"], O.set_(np.zeros(orc["R"].shape), 3.25, O.nz_mask(orc["R"]))))


def test_fig5_program(env):
    """P194-198 (Fig. 5) through the ABI, reading R2: A = 1; B = -1; C = 0.5 A.B -> -10.0."""
    tt, torch = env
    ctx = new_ctx(tt, torch)
    N, M, K = tt.IndexSpace(100), tt.IndexSpace(30), tt.IndexSpace(20)
    tN, tM, tK = tt.TiledIndexSpace(N, 10), tt.TiledIndexSpace(M, sizes=[10, 20]), tt.TiledIndexSpace(K, 5)
    A, B, C = tt.Tensor(ctx, [tM, tK]), tt.Tensor(ctx, [tK, tN]), tt.Tensor(ctx, [tM, tN])
    bufs = [torch.full((T.packed_elems,), float("nan"), dtype=torch.float64, device="cuda") for T in (A, B, C)]
    for T, b in zip((A, B, C), bufs):
        T.bind(b)
    tt.set_(ctx, A, 1.0)
    tt.set_(ctx, B, 0.0)
    J = tt.Tensor(ctx, [tK, tN])
    jb = torch.ones(J.packed_elems, dtype=torch.float64, device="cuda")
    J.bind(jb)
    tt.add(ctx, B, "la", 1.0, -1.0, J, "la")
    tt.contract(ctx, C, "ia", 0.0, 0.5, A, "il", B, "la")
    got = C.download()
    ctx.sync()
    assert np.all(got[:3000] == -10.0)


def test_config2_full_size_sampled(env):
    """BASELINE configs[1] (the bench workload: ladder O=40 V=200 tile 40) at full size, in the
    bench launch configuration: 200 sampled outputs (every C block) vs the oracle element by element
    (K = 40000 each), then a Freivalds check of every output block (inputs regenerated on the host
    by the seeded generator)."""
    tt, torch = env
    pb = ccsd_problem(40, 200, 40, 40, False, terms=("ladder",))
    ctx = new_ctx(tt, torch)
    P = product_objects(tt, ctx, pb)
    bufs = {}
    for name, tag in (("R", 3), ("Vv", 4), ("T", 5)):
        bufs[name] = torch.empty(P[name].packed_elems, dtype=torch.float64, device="cuda")
        P[name].bind(bufs[name])
        tt.fill_synthetic(ctx, P[name], 11, tag)
    tt.contract(ctx, P["R"], "abij", 1.0, 1.0, P["Vv"], "abcd", P["T"], "cdij")
    got = P["R"].download()
    ctx.sync()
    orc = oracle_objects(pb)
    R = orc["R"]
    rng = np.random.default_rng(0)
    idx = []
    for b in range(R.nblocks()):        # 8 per block: 4 corners + 4 random
        o, e = R.block_origin(b), R.block_extents(b)
        corners = [[o[d] + (e[d] - 1 if (q >> d) & 1 else 0) for d in range(4)] for q in (0, 3, 12, 15)]
        idx += corners + [[o[d] + rng.integers(e[d]) for d in range(4)] for _ in range(4)]
    idx = np.array(idx)
    ext = dict(a=200, b=200, c=200, d=200, i=40, j=40)
    sums = O.sampled_elements(idx, "abij", "abcd", "cdij", ext,
                              lambda ix: S.values(11, 4, S.linear_index((200,) * 4, ix)),
                              lambda ix: S.values(11, 5, S.linear_index((200, 200, 40, 40), ix)))
    c0 = S.values(11, 3, S.linear_index((200, 200, 40, 40), idx))
    ref = c0 + sums
    # packed position of each sampled element
    offs = R.blk_off()
    pos = []
    for x in idx:
        b = R.block_id([x[d] // 40 for d in range(4)])
        loc = [x[d] % 40 for d in range(4)]
        pos.append(offs[b] + ((loc[0] * 40 + loc[1]) * 40 + loc[2]) * 40 + loc[3])
    g = got[np.array(pos)]
    assert np.abs(g - ref).max() / np.abs(ref).max() <= TOL
    # Freivalds over every output block: all 1.6e6 x 25 outputs, not samples
    n = np.arange(200, dtype=np.int64)
    t_sub = S.values(11, 5, ((n[:, None, None, None] * 200 + n[None, :, None, None]) * 40
                             + np.arange(40)[None, None, :, None]) * 40 + np.arange(40)[None, None, None, :])
    worst = 0.0
    for b in range(R.nblocks()):
        o = R.block_origin(b)
        ra, rb = np.arange(o[0], o[0] + 40), np.arange(o[1], o[1] + 40)
        v_sub = S.values(11, 4, ((ra[:, None, None, None] * 200 + rb[None, :, None, None]) * 200
                                 + n[None, None, :, None]) * 200 + n[None, None, None, :])
        c0 = S.values(11, 3, ((ra[:, None, None, None] * 200 + rb[None, :, None, None]) * 40
                              + np.arange(40)[None, None, :, None]) * 40 + np.arange(40)[None, None, None, :])
        c_blk = got[offs[b]:offs[b] + 40 ** 4].reshape(40, 40, 40, 40)
        x = rng.uniform(-1.0, 1.0, (40, 40))
        lhs, rhs = O.freivalds(c_blk, "abij", v_sub, "abcd", t_sub, "cdij", x, 1.0, 1.0, c0)
        worst = max(worst, float(np.abs(lhs - rhs).max() / np.abs(rhs).max()))
    assert worst <= TOL, worst


@pytest.mark.parametrize("a_lbl", ["abij", "ijab", "aibj", "jiba", "bajI".replace("I", "i")])
def test_add_modes(env, a_lbl):
    """tt_add in its three element modes (contiguous / multiply-high decode / 32x32 smem transpose)
    on ragged spin-sparse blocks, with zero A blocks read as zeros (S216); scalar on the same pair."""
    tt, torch = env
    spaces = {"O": SpaceSpec(14, tile=5, spin_split=True), "V": SpaceSpec(46, tile=9, spin_split=True)}
    ls = {"a": "V", "b": "V", "i": "O", "j": "O"}
    perm = [a_lbl.index(x) for x in "abij"]        # A dim of each C dim
    c_rule = ("spin", [0, 1], [2, 3])
    a_rule = ("spin", [perm[0], perm[1]], [perm[2], perm[3]])
    pb = Problem(spaces, ls, {"C": TensorSpec("abij", c_rule), "A": TensorSpec(a_lbl, a_rule)})
    ctx = new_ctx(tt, torch)
    orc = oracle_objects(pb)
    P = product_objects(tt, ctx, pb)
    dense = {n: O.dense_masked(orc[n], S.dense(orc[n].shape, 9, t)) for n, t in (("C", 3), ("A", 1))}
    # knock out some A blocks (explicitly zero) to exercise the y_off = -1 path
    bufs = {n: bind_host(torch, P[n], O.pack(orc[n], dense[n])) for n in ("C", "A")}
    for beta in (1.0, 0.0, -0.5):
        tt.add(ctx, P["C"], "abij", beta, 0.75, P["A"], a_lbl)
        got = P["C"].download()
        ctx.sync()
        ref = O.add(dense["C"], "abij", dense["A"], a_lbl, 0.75, beta, cmask=O.nz_mask(orc["C"]))
        assert normwise(got, O.pack(orc["C"], ref)) <= 1e-15
        dense["C"] = ref
    s = tt.contract_scalar(ctx, -0.5, P["A"], a_lbl, P["C"], "abij")
    so = O.scalar(dense["A"], a_lbl, dense["C"], "abij", -0.5)
    assert abs(s - so) <= 1e-13 * max(abs(so), 1.0)


def test_add_zero_input_blocks(env):
    """Explicit nz maps: C blocks whose A block is zero get C = beta*C."""
    tt, torch = env
    spaces = {"X": SpaceSpec(10, tile=4)}
    ls = {"p": "X", "q": "X"}
    nzC = [1, 1, 1, 1, 1, 1, 0, 1, 1]
    nzA = [1, 0, 1, 0, 0, 1, 1, 1, 0]
    pb = Problem(spaces, ls, {"C": TensorSpec("pq", ("nz", nzC)), "A": TensorSpec("pq", ("nz", nzA))})
    ctx = new_ctx(tt, torch)
    orc = oracle_objects(pb)
    P = product_objects(tt, ctx, pb)
    dense = {n: O.dense_masked(orc[n], S.dense(orc[n].shape, 2, t)) for n, t in (("C", 3), ("A", 1))}
    bufs = {n: bind_host(torch, P[n], O.pack(orc[n], dense[n])) for n in ("C", "A")}
    for al in ("pq", "qp"):
        tt.add(ctx, P["C"], "pq", 2.0, 1.0, P["A"], al)
        got = P["C"].download()
        ctx.sync()
        dense["C"] = O.add(dense["C"], "pq", dense["A"], al, 1.0, 2.0, cmask=O.nz_mask(orc["C"]))
        assert normwise(got, O.pack(orc["C"], dense["C"])) <= 1e-15


def _split_all(T, nparts):
    """row parts of every non-zero block of T (all owned by rank 0): exercises the part paths of the
    kernels (row / column offsets of C groups, element ranges of the element ops) on one GPU."""
    parts = []
    for blk in range(T.nblocks):
        if not T.nz[blk]:
            continue
        e0 = int(T.dims[0].offsets[np.unravel_index(blk, T.grid)[0] + 1] - T.dims[0].offsets[np.unravel_index(blk, T.grid)[0]])
        cuts = sorted(set([0, e0] + [e0 * k // nparts for k in range(1, nparts)]))
        parts += [(blk, lo, hi, 0) for lo, hi in zip(cuts[:-1], cuts[1:])]
    T.set_parts(parts)


@pytest.mark.parametrize("k", [0, 1, 2])
def test_row_split_parts_single_rank(env, k):
    """C owned by row parts (all on rank 0) gives bitwise the same contraction as whole blocks;
    set / add / scalar / fill on split tensors match the oracle."""
    tt, torch = env
    pb = ccsd_problem(24, 80, 12, 20, True)
    op = pb.ops[k]
    ctx = new_ctx(tt, torch)
    g1, ref, _, _ = run_contract(tt, torch, ctx, pb, op, alpha=0.5, beta=1.0, seed=4)
    ctx2 = new_ctx(tt, torch)
    C, cl, a, al, b, bl = op
    orc = oracle_objects(pb)
    P = product_objects(tt, ctx2, pb)
    _split_all(P[C], 3)
    assert P[C].parts and all(o == tt.TT_SPLIT for x, o in enumerate(P[C].owner) if P[C].nz[x])
    dense = {}
    bufs = []
    for name, tag in ((C, 3), (a, 1), (b, 2)):
        dense[name] = O.dense_masked(orc[name], S.dense(orc[name].shape, 4, tag))
        bufs.append(bind_host(torch, P[name], O.pack(orc[name], dense[name])))
    tt.contract(ctx2, P[C], cl, 1.0, 0.5, P[a], al, P[b], bl)
    g2 = P[C].download()
    ctx2.sync()
    assert np.array_equal(g1, g2)
    assert normwise(g2, ref) <= TOL
    # element ops on the split tensor
    tt.set_(ctx2, P[C], 0.25)
    got = P[C].download()
    ctx2.sync()
    assert np.array_equal(got, O.pack(orc[C], O.set_(np.zeros(orc[C].shape), 0.25, O.nz_mask(orc[C]))))
    tt.fill_synthetic(ctx2, P[C], 8, 3)
    got = P[C].download()
    ctx2.sync()
    assert np.array_equal(got, O.pack(orc[C], S.dense(orc[C].shape, 8, 3)))


def test_row_split_add_scalar_single_rank(env):
    tt, torch = env
    pb = ccsd_problem(8, 12, 2, 3, True)
    pb.tensors["Rt"] = TensorSpec("ijab", ("spin", [0, 1], [2, 3]))
    ctx = new_ctx(tt, torch)
    orc = oracle_objects(pb)
    P = product_objects(tt, ctx, pb)
    _split_all(P["R"], 2)
    _split_all(P["Ta"], 3)
    dense = {}
    bufs = []
    for name, tag in (("R", 3), ("Rt", 1), ("Ta", 2)):
        dense[name] = O.dense_masked(orc[name], S.dense(orc[name].shape, 3, tag))
        bufs.append(bind_host(torch, P[name], O.pack(orc[name], dense[name])))
    for al in ("ijab", ):
        tt.add(ctx, P["R"], "abij", -0.5, 2.0, P["Rt"], al)
        got = P["R"].download()
        ctx.sync()
        dense["R"] = O.add(dense["R"], "abij", dense["Rt"], al, 2.0, -0.5, cmask=O.nz_mask(orc["R"]))
        assert normwise(got, O.pack(orc["R"], dense["R"])) <= 1e-15
    tt.add(ctx, P["R"], "abij", 1.0, 1.0, P["Ta"], "abij")
    got = P["R"].download()
    ctx.sync()
    dense["R"] = O.add(dense["R"], "abij", dense["Ta"], "abij", 1.0, 1.0, cmask=O.nz_mask(orc["R"]))
    assert normwise(got, O.pack(orc["R"], dense["R"])) <= 1e-15
    for bl in ("acik", "abij"):
        s = tt.contract_scalar(ctx, 0.25, P["Ta"], "acik", P["R"], bl.replace("abij", "acik"))
        so = O.scalar(dense["Ta"], "acik", dense["R"], "acik", 0.25)
        assert abs(s - so) <= 1e-13 * max(abs(so), 1.0)


@pytest.mark.parametrize("labels", [("jbia", "kcai", "bjck"), ("abij", "iack", "kcjb")])
def test_row_split_column_side(env, labels):
    """Row parts of C whose dim-0 label comes from B (the split becomes an n range) or from A."""
    tt, torch = env
    cl, al, bl = labels
    spaces = {"X": SpaceSpec(12, tile=4), "Y": SpaceSpec(10, tile=6), "Z": SpaceSpec(14, tile=8)}
    ls = {"a": "X", "b": "Y", "c": "Z", "i": "Y", "j": "X", "k": "Z"}
    pb = Problem(spaces, ls, {"C": TensorSpec(cl), "A": TensorSpec(al), "B": TensorSpec(bl)}, [("C", cl, "A", al, "B", bl)])
    ctx = new_ctx(tt, torch)
    orc = oracle_objects(pb)
    P = product_objects(tt, ctx, pb)
    _split_all(P["C"], 3)
    dense = {n: O.dense_masked(orc[n], S.dense(orc[n].shape, 6, t)) for n, t in (("C", 3), ("A", 1), ("B", 2))}
    bufs = [bind_host(torch, P[n], O.pack(orc[n], dense[n])) for n in ("C", "A", "B")]
    tt.contract(ctx, P["C"], cl, 0.5, 1.0, P["A"], al, P["B"], bl)
    got = P["C"].download()
    ctx.sync()
    ref = O.contract(dense["C"], cl, dense["A"], al, dense["B"], bl, 1.0, 0.5)
    assert normwise(got, O.pack(orc["C"], ref)) <= TOL


def _cholesky_problem(O_, V_, tO, tV, NL, tL, spin):
    pb = ccsd_problem(O_, V_, tO, tV, spin, terms=("ladder",))
    pb.spaces["L"] = SpaceSpec(NL, tile=tL)
    pb.label_space["L"] = "L"
    pb.tensors["X"] = TensorSpec("acL", ("spin", [0], [1]) if spin else None)
    del pb.tensors["Vv"]
    return pb


@pytest.mark.parametrize("spin,ws_rows,mode", [(True, 1, "bh"), (True, 100, "bh"), (False, 2, "bh"),
                                                (True, 1, "env"), (False, 2, "env"), (True, 3, "auto"),
                                                (True, 2, "densex"), (True, 100, "nobst"), (True, 100, "bst")])
def test_contract_cholesky(env, spin, ws_rows, mode):
    """Implicit Eq. cc12 operand (NEXT-1): R(abij) = beta*R + alpha*sum V(abcd) T(cdij) with V built
    batch by batch from X in a small workspace == oracle with V formed explicitly.  mode "bh": the
    workspace holds the r_t <= s_t half of Bm = T - T(c<->d); "env"/"auto": the two-pass consume
    (forced, or because the workspace holds only W rows); "densex": alpha/beta spaces with a DENSE X map
    (the W / V block maps must follow X's actual map, not the tiles' spins: ADVICE r1).  A roomy
    workspace may also hold BsT (the exchange consume on TMA); "bst" / "nobst": forced on / off
    (TT_CHOL_BST=1 / 0; off = the cp.async exchange consume)."""
    tt, torch = env
    pb = _cholesky_problem(8, 12, 2, 3, 10, 5, spin) if spin else _cholesky_problem(5, 9, 3, 4, 7, 4, False)
    if mode == "densex":
        pb.tensors["X"] = TensorSpec("acL", None)
    if mode == "env":
        os.environ["TT_CHOL_TWO_PASS"] = "1"
    if mode in ("nobst", "bst"):
        os.environ["TT_CHOL_BST"] = "0" if mode == "nobst" else "1"
    ctx = new_ctx(tt, torch)
    orc = oracle_objects(pb)
    P = product_objects(tt, ctx, pb)
    dense, bufs = {}, []
    for name, tag in (("R", 3), ("T", 5), ("X", 7)):
        dense[name] = O.dense_masked(orc[name], S.dense(orc[name].shape, 2, tag))
        bufs.append(bind_host(torch, P[name], O.pack(orc[name], dense[name])))
    tv = max(np.diff(P["X"].dims[0].offsets))
    row = tv ** 4 * P["X"].dims[0].ntiles ** 2 + 64
    bm = 0 if mode == "auto" else P["T"].packed_elems + 32
    if mode == "densex":
        row *= 4
    ws = torch.empty(int(bm + ws_rows * row), dtype=torch.float64, device="cuda")
    for beta in (1.0, 0.0):
        tt.contract_cholesky(ctx, P["R"], "abij", beta, 0.5, P["X"], "abcd", P["T"], "cdij", ws)
        os.environ.pop("TT_CHOL_TWO_PASS", None)
        os.environ.pop("TT_CHOL_BST", None)
        got = P["R"].download()
        ctx.sync()
        st = ctx.stats()
        assert st["aux_flops"] > 0 and st["flops"] > 0
        Vx = O.cholesky_v(dense["X"])
        ref = O.contract(dense["R"], "abij", Vx, "abcd", dense["T"], "cdij", 0.5, beta, cmask=O.nz_mask(orc["R"]))
        assert normwise(got, O.pack(orc["R"], ref)) <= TOL
        dense["R"] = ref


def test_config3_full_size_sampled(env):
    """BASELINE configs[2] at full size (O=60 V=400 tO=30 tV=40, alpha/beta maps; V is 76.8 GB):
    the three doubles terms accumulated into R as bench.py --config cfg3 runs them; 8 sampled outputs
    per non-zero R block (4 corners + 4 random) vs the oracle element by element, zero blocks masked."""
    tt, torch = env
    pb = ccsd_problem(60, 400, 30, 40, True)
    ctx = new_ctx(tt, torch)
    P = product_objects(tt, ctx, pb)
    orc = oracle_objects(pb)
    tags = {"R": 3, "Vv": 4, "T": 5, "Ta": 1, "Wr": 2, "Tb": 6, "Wh": 7}
    bufs = {}
    for name in pb.tensors:
        bufs[name] = torch.empty(P[name].packed_elems, dtype=torch.float64, device="cuda")
        P[name].bind(bufs[name])
        tt.fill_synthetic(ctx, P[name], 13, tags[name])
    for (c, cl, a, al, b, bl) in pb.ops:
        tt.contract(ctx, P[c], cl, 1.0, 1.0, P[a], al, P[b], bl)
    got = P["R"].download()
    ctx.sync()
    del bufs
    torch.cuda.empty_cache()
    R = orc["R"]
    rng = np.random.default_rng(1)
    idx = []
    for blk in range(R.nblocks()):
        if not R.nz[blk]:
            continue
        o, e = R.block_origin(blk), R.block_extents(blk)
        idx += [[o[d] + (e[d] - 1 if (qq >> d) & 1 else 0) for d in range(4)] for qq in (0, 5, 10, 15)]
        idx += [[o[d] + rng.integers(e[d]) for d in range(4)] for _ in range(4)]
    idx = np.array(idx)
    ext = dict(a=400, b=400, c=400, d=400, i=60, j=60, k=60, l=60)

    def gen(name):
        T = orc[name]
        return (lambda ix: S.values(13, tags[name], S.linear_index(T.shape, ix)),
                lambda ix: _nz_elem(T, ix))

    ref = S.values(13, 3, S.linear_index(R.shape, idx))
    for (c, cl, a, al, b, bl) in pb.ops:
        av, anz = gen(a)
        bv, bnz = gen(b)
        ref = ref + O.sampled_elements(idx, cl, al, bl, ext, av, bv, anz, bnz)
    offs = R.blk_off()
    pos = []
    for x in idx:
        blk = R.block_id([int(np.searchsorted(R.dims[d].offsets, x[d], side="right") - 1) for d in range(4)])
        org, e = R.block_origin(blk), R.block_extents(blk)
        loc = [x[d] - org[d] for d in range(4)]
        pos.append(offs[blk] + ((loc[0] * e[1] + loc[1]) * e[2] + loc[2]) * e[3] + loc[3])
    g = got[np.array(pos)]
    assert np.abs(g - ref).max() / np.abs(ref).max() <= TOL


def _nz_elem(T, ix):
    """1 where the global index tuples ix lie in a non-zero block of oracle tensor T."""
    ix = np.asarray(ix)
    tiles = [np.searchsorted(np.asarray(T.dims[d].offsets), ix[..., d], side="right") - 1 for d in range(T.order)]
    bid = np.zeros(ix.shape[:-1], dtype=np.int64)
    for d, g in enumerate(T.grid):
        bid = bid * g + tiles[d]
    return np.asarray(T.nz, dtype=np.uint8)[bid]


@pytest.mark.parametrize("variant", [3, 4, 5])
@pytest.mark.parametrize("tv", [20, 24])
def test_tma_producer(env, variant, tv):
    """TMA producer (uniform fused ladder operands; tV=24 gives a ragged last M tile whose extra rows
    read the next block): bitwise equal to the cp.async producer, and the oracle within 1e-11."""
    tt, torch = env
    pb = ccsd_problem(24, 4 * tv, 12, tv, True, terms=("ladder",))
    outs = []
    for tma in ("1", "0"):
        os.environ["TT_TMA"] = tma
        ctx = new_ctx(tt, torch, variant)
        got, ref, _, _ = run_contract(tt, torch, ctx, pb, pb.ops[0], alpha=0.5, beta=1.0, seed=8)
        assert ctx.stats()["producer"] == (1 if tma == "1" else 0)
        assert normwise(got, ref) <= TOL
        outs.append(got)
    os.environ.pop("TT_TMA", None)
    os.environ.pop("TT_FORCE_VARIANT", None)
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["spin_small_ladder", "ragged_dense_ring", "multi_tile_spin_ladder"])
def test_variants_bitwise_equal(env, name):
    """Every tile variant (classic 0-2, warp-specialised 3-5; TMA or cp.async producers) adds each output
    element's products in the same k order and the same groups of four per DMMA step, so they give the
    same bits -- neither the variant model, nor the measured autotuning (TT_AUTOTUNE), nor a different
    partition (row-split parts pick their own variants) changes a result (R12)."""
    tt, torch = env
    pb, k = PROBLEMS[name]
    outs = []
    for v in (0, 1, 2, 3, 4, 5):
        ctx = new_ctx(tt, torch, variant=v)
        got, ref, _, _ = run_contract(tt, torch, ctx, pb, pb.ops[k], seed=3)
        assert normwise(got, ref) <= TOL
        outs.append(got)
    os.environ.pop("TT_FORCE_VARIANT", None)
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


def _vec_problem(spin):
    spaces = {"O": SpaceSpec(6, tile=2, spin_split=spin), "V": SpaceSpec(10, tile=3, spin_split=spin),
              "L": SpaceSpec(23, tile=7)}
    ls = {"f": "V", "a": "V", "e": "V", "m": "O", "i": "O", "L": "L"}
    sp = (lambda up, lo: ("spin", up, lo)) if spin else (lambda up, lo: None)
    tensors = {"T1": TensorSpec("fm", sp([0], [1])), "Xov": TensorSpec("mfL", sp([0], [1])),
               "g": TensorSpec("L"), "X": TensorSpec("aeL", sp([0], [1])), "F": TensorSpec("ae", sp([0], [1])),
               "Xvo": TensorSpec("aiL", sp([0], [1])), "R1": TensorSpec("ai", sp([0], [1]))}
    ops = [("g", "L", "T1", "fm", "Xov", "mfL"),       # A without free labels: M = 1
           ("F", "ae", "X", "aeL", "g", "L"),          # B without free labels: N = 1
           ("R1", "ai", "g", "L", "Xvo", "aiL")]       # A without free labels, K = 1 group
    return Problem(spaces, ls, tensors, ops)


@pytest.mark.parametrize("spin", [False, True])
@pytest.mark.parametrize("k", [0, 1, 2])
def test_vector_shaped_contractions(env, spin, k):
    """Matrix-vector shapes of the Cholesky-factorized CCSD terms (g(L) = sum_mf t_m^f X(m,f,L),
    F(a,e) += sum_L X(a,e,L) g(L)): an operand or the output without free labels on one GEMM side."""
    tt, torch = env
    pb = _vec_problem(spin)
    ctx = new_ctx(tt, torch)
    got, ref, _, _ = run_contract(tt, torch, ctx, pb, pb.ops[k], alpha=0.5, beta=1.0)
    assert normwise(got, ref) <= TOL, normwise(got, ref)


@pytest.mark.parametrize("terms", [("ladder",), ("ring",), ("ladder", "ring", "hh")])
def test_contract_host_bitwise(env, terms):
    """tt_contract_host (host buffers, pipelined per dim-0 tile inside the library) gives bitwise the
    result of upload + tt_contract + download, and the oracle's within 1e-11."""
    tt, torch = env
    pb = ccsd_problem(12, 30, 3, 7, True, terms=terms)
    orc = oracle_objects(pb)
    ctx = new_ctx(tt, torch)
    P = product_objects(tt, ctx, pb)
    host, dense, dev = {}, {}, {}
    for i, name in enumerate(sorted(orc)):
        dense[name] = O.dense_masked(orc[name], S.dense(orc[name].shape, 4, 1 + i))
        host[name] = torch.from_numpy(O.pack(orc[name], dense[name])).pin_memory()
        dev[name] = torch.zeros(P[name].storage_elems, dtype=torch.float64, device="cuda")
        P[name].bind(dev[name])
    out = host["R"].clone().pin_memory()
    ref_d = dense["R"]
    for k, (c, cl, a, al, b, bl) in enumerate(pb.ops):
        tt.contract_host(ctx, P[c], cl, 1.0, 0.5, P[a], al, P[b], bl, host[a], host[b], out,
                         c_in=(k == 0), c_out=(k == len(pb.ops) - 1))
        ref_d = O.contract(ref_d, cl, dense[a], al, dense[b], bl, 0.5, 1.0, cmask=O.nz_mask(orc[c]))
    ctx.sync()
    got = out.numpy().copy()
    # plain path on a second context
    ctx2 = new_ctx(tt, torch)
    P2 = product_objects(tt, ctx2, pb)
    keep = {}
    for name in orc:
        keep[name] = host[name].cuda()
        P2[name].bind(keep[name])
    for (c, cl, a, al, b, bl) in pb.ops:
        tt.contract(ctx2, P2[c], cl, 1.0, 0.5, P2[a], al, P2[b], bl)
    plain = P2["R"].download()
    ctx2.sync()
    assert np.array_equal(got, plain)
    ref = O.pack(orc["R"], ref_d)
    assert normwise(got, ref) <= TOL


def _wbuild_problem(n, tv, NL, tl, spin):
    spaces = {"V": SpaceSpec(n, tile=tv, spin_split=spin), "L": SpaceSpec(NL, tile=tl)}
    sp = (lambda up, lo: ("spin", up, lo)) if spin else (lambda up, lo: None)
    return Problem(spaces, {"p": "V", "q": "V", "r": "V", "s": "V", "L": "L"},
                   {"W": TensorSpec("pqrs", sp([0, 1], [2, 3])), "X": TensorSpec("prL", sp([0], [1])),
                    "Y": TensorSpec("qsL", sp([0], [1]))},
                   [("W", "pqrs", "X", "prL", "Y", "qsL")])


@pytest.mark.parametrize("variant", [3, 4, 5])
@pytest.mark.parametrize("case", ["wbuild_ktail", "wbuild_k16", "ladder_ktail", "hh_ktail"])
def test_tma_general_layouts(env, variant, case):
    """TMA producer beyond the uniform ladder: [N][K] B operands with a permuted (multi-group) output --
    the implicit operand's W(p,q,r,s) = X(p,r,L) X(q,s,L) -- and K extents that are not multiples of 16
    (the k tail is TMA out-of-bounds zero fill: a [blocks][K][N] view for [K][N] operands).  Bitwise
    equal to the cp.async producer and within 1e-11 of the oracle."""
    tt, torch = env
    if case == "wbuild_ktail":
        pb, beta = _wbuild_problem(20, 5, 20, 10, True), 0.0        # K = L tile 10: a tail of 10
    elif case == "wbuild_k16":
        pb, beta = _wbuild_problem(24, 6, 64, 32, False), 0.0
    elif case == "ladder_ktail":
        pb, beta = ccsd_problem(12, 24, 6, 6, True, terms=("ladder",)), 1.0   # K = 36: tail of 4
    else:
        pb, beta = ccsd_problem(12, 12, 6, 6, False, terms=("hh",)), 1.0      # K = 36
    outs = []
    for tma in ("1", "0"):
        os.environ["TT_TMA"] = tma
        ctx = new_ctx(tt, torch, variant)
        got, ref, _, _ = run_contract(tt, torch, ctx, pb, pb.ops[0], alpha=0.5, beta=beta, seed=9)
        assert ctx.stats()["producer"] == (1 if tma == "1" else 0), case
        assert normwise(got, ref) <= TOL
        outs.append(got)
    os.environ.pop("TT_TMA", None)
    os.environ.pop("TT_FORCE_VARIANT", None)
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("name", ["multi_tile_spin_ring", "ragged_dense_ring", "ragged_dense_ladder"])
@pytest.mark.parametrize("variant", [3, 4])
def test_wave_tail_split_bitwise(env, name, variant):
    """The wave tail (the last work items re-tiled with the smallest warp-specialised tile and launched
    after the main kernel; TT_TAIL_SLOTS forces it on small plans) gives bitwise the C of the unsplit
    plan, on the TMA and the cp.async producer, and the oracle's within 1e-11."""
    tt, torch = env
    pb, k = PROBLEMS[name]
    out, launches = {}, {}
    try:
        for mode in ("off", "on"):
            os.environ["TT_TAIL_SPLIT"] = "0" if mode == "off" else "1"
            if mode == "on":   # a slot count that leaves a partial last wave
                w = out["work_items"]
                os.environ["TT_TAIL_SLOTS"] = str(next(x for x in (7, 5, 11, 13, 3, 2) if w > x and w % x))
            ctx = new_ctx(tt, torch, variant=variant)
            ctx.set_profiling(True)
            got, ref, _, _ = run_contract(tt, torch, ctx, pb, pb.ops[k], alpha=0.5, beta=1.0)
            launches[mode] = ctx.profile("tt_contract_dmma")[1]
            out["work_items"] = ctx.stats()["work_items"]
            out[mode] = got
            assert normwise(got, ref) <= TOL
    finally:
        for e in ("TT_TAIL_SPLIT", "TT_TAIL_SLOTS", "TT_FORCE_VARIANT"):
            os.environ.pop(e, None)
    assert launches["off"] == 1 and launches["on"] == 2, launches
    assert np.array_equal(out["on"], out["off"])
