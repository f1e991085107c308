"""Scheduler (P178, P191-199, P215; reading R25): levelization on the host (CPU) and execution on
the GPU (concurrent streams per level == sequential immediate execution, bitwise)."""
import numpy as np
import pytest

import paper_2201_01257_b200 as tt
import synthetic as S
from oracle import ops as O
from oracle import sched as OS
from tests.cases import TensorSpec, ccsd_problem, oracle_objects, product_objects


def _fig5(ctx):
    N, M, K = tt.IndexSpace(100), tt.IndexSpace(30), tt.IndexSpace(20)
    tN, tM, tK = tt.TiledIndexSpace(N, 10), tt.TiledIndexSpace(M, sizes=[10, 20]), tt.TiledIndexSpace(K, 5)
    A, B, C, J = tt.Tensor(ctx, [tM, tK]), tt.Tensor(ctx, [tK, tN]), tt.Tensor(ctx, [tM, tN]), tt.Tensor(ctx, [tK, tN])
    return (N, M, K, tN, tM, tK), A, B, C, J


def test_fig5_three_levels():
    """S470: Fig. 5 (set A; B += -1*...(A); C = 0.5 A.B) -> levels {set}, {add}, {mult}."""
    ctx = tt.Context(device=-1)
    keep, A, B, C, J = _fig5(ctx)
    s = tt.Scheduler(ctx)
    s.set_(A, 1.0).add(B, "la", 1.0, -1.0, J, "la").contract(C, "ia", 0.0, 0.5, A, "il", B, "la")
    lv, L = s.levels()
    assert lv == [0, 0, 1] and L == 2       # with reading R2 the add does not read A
    s2 = tt.Scheduler(ctx)
    s2.set_(A, 1.0).add(B, "la", 1.0, -1.0, A, "la").contract(C, "ia", 0.0, 0.5, A, "il", B, "la")
    assert s2.levels() == ([0, 1, 2], 3)    # as printed (add reads A): three levels, S470


@pytest.mark.parametrize("seed", range(12))
def test_levels_match_oracle_and_longest_chain(seed):
    rng = np.random.default_rng(seed)
    ctx = tt.Context(device=-1)
    sp = tt.IndexSpace(8)
    t4 = tt.TiledIndexSpace(sp, 4)
    T = [tt.Tensor(ctx, [t4, t4]) for _ in range(5)]
    s = tt.Scheduler(ctx)
    ops = []
    res = []
    for _ in range(int(rng.integers(1, 11))):
        kind = int(rng.integers(0, 4))
        c, a, b = (int(x) for x in rng.choice(5, 3, replace=False))
        beta = float(rng.integers(0, 2))
        if kind == 0:
            s.set_(T[c], 1.0)
            ops.append((set(), {c}))
        elif kind == 1:
            s.add(T[c], "ij", beta, 1.0, T[a], "ji")
            ops.append(({a} | ({c} if beta else set()), {c}))
        elif kind == 2:
            s.contract(T[c], "ij", beta, 1.0, T[a], "ik", T[b], "kj")
            ops.append(({a, b} | ({c} if beta else set()), {c}))
        else:
            s.scalar(1.0, T[a], "ij", T[b], "ij")
            ops.append(({a, b}, set()))
    lv, L = s.levels()
    assert lv == OS.levelize(ops)
    assert L == OS.longest_chain_bruteforce(ops)
    for i in range(len(ops)):
        for j in range(i):
            if lv[i] == lv[j]:
                assert not OS.conflicts(ops[i], ops[j])


def test_host_only_cannot_execute():
    ctx = tt.Context(device=-1)
    keep, A, B, C, J = _fig5(ctx)
    s = tt.Scheduler(ctx)
    s.set_(A, 1.0)
    with pytest.raises(tt.TTError) as e:
        s.execute()
    assert e.value.name == "TT_E_STATE"


@pytest.mark.gpu
def test_sched_fig5_gpu():
    import torch
    ctx = tt.Context(device=0, stream=torch.cuda.current_stream().cuda_stream)
    keep, A, B, C, J = _fig5(ctx)
    bufs = [torch.full((T.packed_elems,), float("nan"), dtype=torch.float64, device="cuda") for T in (A, B, C)]
    for T, b in zip((A, B, C), bufs):
        T.bind(b)
    jb = torch.ones(J.packed_elems, dtype=torch.float64, device="cuda")
    J.bind(jb)
    s = tt.Scheduler(ctx, nstreams=3)
    s.set_(A, 1.0).set_(B, 0.0).add(B, "la", 1.0, -1.0, J, "la").contract(C, "ia", 0.0, 0.5, A, "il", B, "la")
    assert s.levels() == ([0, 0, 1, 2], 3)
    s.execute()
    got = C.download()
    ctx.sync()
    assert np.all(got[:3000] == -10.0)
    assert s.stats()["levels_executed"] == 3


@pytest.mark.gpu
def test_sched_matches_sequential_bitwise():
    """A CCSD-shaped mini program with independent ops in each level: the scheduled run (concurrent
    streams) is bitwise equal to immediate sequential calls and to the oracle within 1e-11."""
    import torch
    pb = ccsd_problem(8, 12, 2, 3, True)
    pb.tensors["R2"] = TensorSpec("abij", ("spin", [0, 1], [2, 3]))
    pb.tensors["R3"] = TensorSpec("abij", ("spin", [0, 1], [2, 3]))
    stream = torch.cuda.current_stream().cuda_stream
    outs = []
    for mode in ("sched", "seq"):
        ctx = tt.Context(device=0, stream=stream)
        orc = oracle_objects(pb)
        P = product_objects(tt, ctx, pb)
        bufs = []
        dense = {}
        for i, name in enumerate(sorted(pb.tensors)):
            dense[name] = O.dense_masked(orc[name], S.dense(orc[name].shape, 4, i + 1))
            b = torch.from_numpy(O.pack(orc[name], dense[name])).cuda()
            P[name].bind(b)
            bufs.append(b)
        prog = [
            ("contract", "R", "abij", 1.0, 1.0, "Vv", "abcd", "T", "cdij"),     # level 0
            ("contract", "R2", "abij", 0.0, 0.5, "Ta", "acik", "Wr", "cbkj"),   # level 0
            ("contract", "R3", "abij", 1.0, -1.0, "Tb", "abkl", "Wh", "klij"),  # level 0
            ("add", "R", "abij", 1.0, 1.0, "R2", "abij"),                       # level 1
            ("add", "R3", "abij", 2.0, 1.0, "R2", "baji"),                      # level 1
            ("scalar", 0.25, "R", "abij", "R3", "abij"),                        # level 2
        ]
        res = []
        if mode == "sched":
            s = tt.Scheduler(ctx, nstreams=3)
            for op in prog:
                if op[0] == "contract":
                    s.contract(P[op[1]], op[2], op[3], op[4], P[op[5]], op[6], P[op[7]], op[8])
                elif op[0] == "add":
                    s.add(P[op[1]], op[2], op[3], op[4], P[op[5]], op[6])
                else:
                    s.scalar(op[1], P[op[2]], op[3], P[op[4]], op[5])
            assert s.levels() == ([0, 0, 0, 1, 1, 2], 3)
            res = s.execute()
        else:
            for op in prog:
                if op[0] == "contract":
                    tt.contract(ctx, P[op[1]], op[2], op[3], op[4], P[op[5]], op[6], P[op[7]], op[8])
                elif op[0] == "add":
                    tt.add(ctx, P[op[1]], op[2], op[3], op[4], P[op[5]], op[6])
                else:
                    res.append(tt.contract_scalar(ctx, op[1], P[op[2]], op[3], P[op[4]], op[5]))
        outs.append(([P[n].download() for n in ("R", "R2", "R3")], res))
        ctx.sync()
    (a, ra), (b, rb) = outs
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert ra == rb
    # oracle
    m = O.nz_mask(orc["R"])
    R = O.contract(dense["R"], "abij", dense["Vv"], "abcd", dense["T"], "cdij", 1.0, 1.0, cmask=m)
    R2 = O.contract(dense["R2"], "abij", dense["Ta"], "acik", dense["Wr"], "cbkj", 0.5, 0.0, cmask=m)
    R3 = O.contract(dense["R3"], "abij", dense["Tb"], "abkl", dense["Wh"], "klij", -1.0, 1.0, cmask=m)
    R = O.add(R, "abij", R2, "abij", 1.0, 1.0, cmask=m)
    R3 = O.add(R3, "abij", R2, "baji", 1.0, 2.0, cmask=m)
    E = O.scalar(R, "abij", R3, "abij", 0.25)
    ref = O.pack(orc["R"], R)
    assert np.abs(a[0] - ref).max() / np.abs(ref).max() <= 1e-11
    assert abs(ra[0] - E) <= 1e-12 * abs(E)


@pytest.mark.gpu
def test_sched_graph_replay_bitwise():
    """CUDA-graph capture of a queue (plans built first, levels with forked streams recorded) and two
    replays == running the same program twice with immediate calls, bitwise; scalar results too."""
    import torch
    pb = ccsd_problem(8, 12, 2, 3, True)
    pb.tensors["R2"] = TensorSpec("abij", ("spin", [0, 1], [2, 3]))
    stream = torch.cuda.current_stream().cuda_stream
    outs = []
    for mode in ("graph", "seq"):
        ctx = tt.Context(device=0, stream=stream)
        orc = oracle_objects(pb)
        P = product_objects(tt, ctx, pb)
        bufs = []
        for i, name in enumerate(sorted(pb.tensors)):
            b = torch.from_numpy(O.pack(orc[name], O.dense_masked(orc[name], S.dense(orc[name].shape, 6, i + 1)))).cuda()
            P[name].bind(b)
            bufs.append(b)
        res = []
        if mode == "graph":
            s = tt.Scheduler(ctx, nstreams=2)
            s.contract(P["R"], "abij", 1.0, 0.5, P["Vv"], "abcd", P["T"], "cdij")
            s.contract(P["R2"], "abij", 0.0, 1.0, P["Ta"], "acik", P["Wr"], "cbkj")
            s.add(P["R"], "abij", 1.0, -1.0, P["R2"], "baji")
            s.scalar(0.25, P["R"], "abij", P["T"], "abij".replace("ab", "ab"))
            s.capture()
            for _ in range(2):
                res += s.replay()
        else:
            for _ in range(2):
                tt.contract(ctx, P["R"], "abij", 1.0, 0.5, P["Vv"], "abcd", P["T"], "cdij")
                tt.contract(ctx, P["R2"], "abij", 0.0, 1.0, P["Ta"], "acik", P["Wr"], "cbkj")
                tt.add(ctx, P["R"], "abij", 1.0, -1.0, P["R2"], "baji")
                res.append(tt.contract_scalar(ctx, 0.25, P["R"], "abij", P["T"], "abij"))
        outs.append((P["R"].download(), P["R2"].download(), res))
        ctx.sync()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]


def test_views_conflict_with_their_parent():
    """A view shares its parent's storage (R29): an op writing a view conflicts with ops reading or
    writing the parent or another view of it (handles alone missed this)."""
    ctx = tt.Context(device=-1)
    sp = tt.IndexSpace(8, [(0, 4), (4, 8)], [1, -1])
    t4 = tt.TiledIndexSpace(sp, 4)
    T, U, W = tt.Tensor(ctx, [t4, t4]), tt.Tensor(ctx, [t4, t4]), tt.Tensor(ctx, [t4, t4])
    first, second = t4(0), t4(1)
    V1 = T.view([first, t4])
    V2 = T.view([second, t4])
    s = tt.Scheduler(ctx)
    s.add(V1, "ij", 0.0, 1.0, U.view([first, t4]), "ij")   # writes T (through V1)
    s.add(W, "ij", 0.0, 1.0, T, "ij")                       # reads the parent
    s.add(V2, "ij", 0.0, 1.0, U.view([second, t4]), "ij")  # writes T again (other view)
    s.scalar(1.0, U, "ij", W, "ij")                         # unrelated to T: reads W (written at level 1)
    assert s.levels() == ([0, 1, 2, 2], 3)


def test_cholesky_workspace_is_a_written_resource():
    """Two implicit-operand contractions on one workspace never share a level (the workspace holds
    each one's W batches); on disjoint workspaces they may."""
    import torch
    ctx = tt.Context(device=-1)
    so, sv, sl = tt.IndexSpace(4), tt.IndexSpace(6), tt.IndexSpace(5)
    to, tv, tl = tt.TiledIndexSpace(so, 2), tt.TiledIndexSpace(sv, 3), tt.TiledIndexSpace(sl, 5)
    X = tt.Tensor(ctx, [tv, tv, tl])
    Tt = tt.Tensor(ctx, [tv, tv, to, to])
    R1, R2 = tt.Tensor(ctx, [tv, tv, to, to]), tt.Tensor(ctx, [tv, tv, to, to])
    ws = torch.empty(1000, dtype=torch.float64)
    for (o1, o2), expect in (((0, 0), [0, 1]), ((0, 500), [0, 0])):
        s = tt.Scheduler(ctx)
        s.contract_cholesky(R1, "abij", 0.0, 1.0, X, "abcd", Tt, "cdij", ws[o1:o1 + 500])
        s.contract_cholesky(R2, "abij", 0.0, 1.0, X, "abcd", Tt, "cdij", ws[o2:o2 + 500])
        assert s.levels()[0] == expect
