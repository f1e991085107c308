"""Multi-rank paths on ONE GPU through simulated ranks: every rank's
partition, owners, gather plan and kernels run unchanged; only the transport is device copies between
the ranks' buffers (and a rank-order scalar sum).  For p in {2, 3, 8}: the ladder, ring and hole-hole
terms (inputs round robin, so each rank gathers what it reads; part of an input row-split), a
permuted add, the row-split output (tt_partition_split), the implicit Cholesky ladder (X replicated,
Bm half all-gathered), and the scalar all-reduce.  Results: tensors assembled from the owned ranges are
BITWISE equal to the p = 1 run (reading R12: one rank computes each element with the full canonical K
sum) and within 1e-11 of the oracle; scalars within 1e-13 (all-reduce order).  Ref: P212 (SPMD, access
to remote portions), S506 (rank invariance)."""
import numpy as np
import pytest

import synthetic as S
from oracle import layout as Lo
from oracle import ops as O
from tests.cases import TensorSpec, ccsd_problem, oracle_objects, product_objects
from tests.simranks import assemble, run_ranks

pytestmark = pytest.mark.gpu

TAGS = (("R", 3), ("Vv", 4), ("T", 5), ("Ta", 1), ("Wr", 2), ("Tb", 6), ("Wh", 7), ("Rt", 8))


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2201_01257_b200 as tt
    torch.cuda.init()
    return tt, torch


def _problem():
    pb = ccsd_problem(12, 24, 3, 6, True)
    pb.tensors["Rt"] = TensorSpec("ijab", ("spin", [0, 1], [2, 3]))
    return pb


def _body(tt, torch, pb, split):
    def body(rank, ctx):
        P = product_objects(tt, ctx, pb)
        c0, cl0, a0, al0, b0, bl0 = pb.ops[0]
        world = ctx.nranks
        if split:
            tt.partition_split(ctx, P[c0], cl0, P[a0], al0, P[b0], bl0, group_dims=(0, 1))
            parts = []
            for blk in range(P["Ta"].nblocks):   # some input rows split across ranks too
                if P["Ta"].nz[blk] and blk % 3 == 0:
                    e0 = int(np.diff(P["Ta"].dims[0].offsets)[np.unravel_index(blk, P["Ta"].grid)[0]])
                    parts += [(blk, 0, e0 // 2, blk % world), (blk, e0 // 2, e0, (blk + 1) % world)]
            P["Ta"].set_parts(parts)
        else:
            P[c0].set_owner(tt.partition_lpt(ctx, P[c0], cl0, P[a0], al0, P[b0], bl0))
        bufs = {}
        for name, tag in TAGS:   # non-held blocks stay NaN: a missed gather poisons the result
            bufs[name] = torch.full((P[name].storage_elems,), float("nan"), dtype=torch.float64, device="cuda")
            P[name].bind(bufs[name])
            tt.fill_synthetic(ctx, P[name], 3, tag)
        for k, (c, cl, a, al, b, bl) in enumerate(pb.ops):
            tt.contract(ctx, P[c], cl, 1.0, 0.5 + k, P[a], al, P[b], bl)
        tt.add(ctx, P["R"], "abij", 1.0, -0.25, P["Rt"], "ijab")
        s = tt.contract_scalar(ctx, 0.25, P["Ta"], "acik", P["R"], "acik")
        # implicit Cholesky ladder: X replicated, R2 row-split on (a,b) rows, T round robin (B gathered)
        so, sv = P["_keep"][1]["O"], P["_keep"][1]["V"]
        tL = tt.TiledIndexSpace(tt.IndexSpace(10), 5)
        X = tt.Tensor(ctx, [sv, sv, tL], spin=([0], [1]))
        X.set_owner(np.where(X.nz > 0, tt.TT_REPLICATED, -1).astype(np.int32))
        R2 = tt.Tensor(ctx, [sv, sv, so, so], spin=([0, 1], [2, 3]))
        tt.partition_split(ctx, R2, "abij", P["Vv"], "abcd", P["T"], "cdij", group_dims=(0, 1))
        xb = torch.empty(X.storage_elems, dtype=torch.float64, device="cuda")
        r2b = torch.full((R2.storage_elems,), float("nan"), dtype=torch.float64, device="cuda")
        X.bind(xb)
        R2.bind(r2b)
        tt.fill_synthetic(ctx, X, 3, 9)
        tt.fill_synthetic(ctx, R2, 3, 10)
        ws = torch.empty(P["T"].packed_elems + 32 + 12 ** 4 * 16, dtype=torch.float64, device="cuda")
        tt.contract_cholesky(ctx, R2, "abij", 1.0, 0.5, X, "abcd", P["T"], "cdij", ws)
        out = {"R": (P["R"], P["R"].download()), "R2": (R2, R2.download()), "s": s}
        ctx.sync()
        return out
    return body


def _oracle(pb):
    orc = oracle_objects(pb)
    dense = {n: O.dense_masked(orc[n], S.dense(orc[n].shape, 3, t)) for n, t in TAGS}
    m = O.nz_mask(orc["R"])
    Rd = dense["R"]
    for k, (c, cl, a, al, b, bl) in enumerate(pb.ops):
        Rd = O.contract(Rd, cl, dense[a], al, dense[b], bl, 0.5 + k, 1.0, cmask=m)
    Rd = O.add(Rd, "abij", dense["Rt"], "ijab", -0.25, 1.0, cmask=m)
    so = O.scalar(dense["Ta"], "acik", Rd, "acik", 0.25)
    oX = Lo.tensor_spin([orc["Vv"].dims[0], orc["Vv"].dims[0], Lo.tile_fixed(Lo.IndexSpace(10), 5)], [0], [1])
    Xd = O.dense_masked(oX, S.dense(oX.shape, 3, 9))
    R2d = O.dense_masked(orc["R"], S.dense(orc["R"].shape, 3, 10))
    R2 = O.contract(R2d, "abij", O.cholesky_v(Xd), "abcd", dense["T"], "cdij", 0.5, 1.0, cmask=m)
    return O.pack(orc["R"], Rd), O.pack(orc["R"], R2), so


_CACHE = {}


def _run(tt, torch, p, split):
    key = (p, split)
    if key not in _CACHE:
        pb = _problem()
        res = run_ranks(tt, torch, p, _body(tt, torch, pb, split))
        R, seen = assemble([r["R"][0] for r in res], [r["R"][1] for r in res], res[0]["R"][0].packed_elems)
        R2, seen2 = assemble([r["R2"][0] for r in res], [r["R2"][1] for r in res], res[0]["R2"][0].packed_elems)
        _CACHE[key] = (R, seen, R2, seen2, [r["s"] for r in res])
    return _CACHE[key]


@pytest.mark.parametrize("split", [True, False])
@pytest.mark.parametrize("p", [2, 3, 8])
def test_simulated_ranks_bitwise_and_oracle(env, p, split):
    tt, torch = env
    R1, seen1, R21, seen21, s1 = _run(tt, torch, 1, split)
    Rp, seenp, R2p, seen2p, sp = _run(tt, torch, p, split)
    assert np.array_equal(seen1, seenp) and np.array_equal(seen21, seen2p)
    assert not np.isnan(Rp[seenp]).any() and not np.isnan(R2p[seen2p]).any()
    assert np.array_equal(Rp[seenp], R1[seen1]), "tensor result depends on the rank count"
    assert np.array_equal(R2p[seen2p], R21[seen21]), "Cholesky ladder depends on the rank count"
    refR, refR2, so = _oracle(_problem())
    errR = np.abs(Rp[seenp] - refR[seenp]).max() / np.abs(refR[seenp]).max()
    errR2 = np.abs(R2p[seen2p] - refR2[seen2p]).max() / np.abs(refR2[seen2p]).max()
    assert errR <= 1e-11 and errR2 <= 1e-11, (errR, errR2)
    assert len(set(sp)) == 1, "ranks disagree on the all-reduced scalar"
    assert abs(sp[0] - so) <= 1e-13 * abs(so) and abs(s1[0] - so) <= 1e-13 * abs(so)


def test_simulated_gather_moves_exactly_the_plan(env):
    """The simulated exchange receives exactly the bytes of the gather plan (tt_last_stats
    gathered_bytes), and a rank with round-robin inputs receives something (the path is exercised)."""
    tt, torch = env
    pb = _problem()

    def body(rank, ctx):
        P = product_objects(tt, ctx, pb)
        c, cl, a, al, b, bl = pb.ops[1]
        bufs = []
        for name in (c, a, b):
            buf = torch.zeros(P[name].storage_elems, dtype=torch.float64, device="cuda")
            P[name].bind(buf)
            bufs.append(buf)
        plan = tt.gather_plan(ctx, P[c], cl, P[a], al, P[b], bl)
        tt.contract(ctx, P[c], cl, 1.0, 1.0, P[a], al, P[b], bl)
        ctx.sync()
        return plan, ctx.stats()["gathered_bytes"]

    res = run_ranks(tt, torch, 3, body)
    for (recv, send), got in res:
        assert len(recv) > 0 and got == int(sum(8 * (e - b) for (_, _, _, b, e) in recv))


def _mirror_rows(tt, C, A):
    """A's (a,b) rows follow C's owner-computes rows (whole blocks or row parts), as bench.py places V."""
    whole, split = {}, {}
    for blk in range(C.nblocks):
        if C.nz[blk] and C.owner[blk] >= 0:
            whole[tuple(int(x) for x in np.unravel_index(blk, C.grid)[:2])] = int(C.owner[blk])
    for (blk, lo, hi, ow) in C.parts:
        split.setdefault(tuple(int(x) for x in np.unravel_index(blk, C.grid)[:2]), set()).add((lo, hi, ow))
    own = np.full(A.nblocks, -1, np.int32)
    parts = []
    for blk in range(A.nblocks):
        if not A.nz[blk]:
            continue
        key = tuple(int(x) for x in np.unravel_index(blk, A.grid)[:2])
        if key in split:
            parts += [(blk, lo, hi, ow) for (lo, hi, ow) in sorted(split[key])]
            own[blk] = 0
        else:
            own[blk] = whole.get(key, 0)
    A.set_owner(own)
    if parts:
        A.set_parts(parts)


@pytest.mark.parametrize("p", [2, 3])
def test_simulated_contract_host_pipelined(env, p):
    """tt_contract_host with several ranks: R row-split on (a,b) rows, V's rows mirrored (local to each
    rank's R rows), T round robin (gathered up front): each rank pipelines its held V rows chunk by chunk
    (several kernel launches), and the R ranges the ranks own, assembled from their host buffers, equal
    bit for bit the 1-rank result, which is within 1e-11 of the oracle."""
    tt, torch = env
    pb = _problem()
    c, cl, a, al, b, bl = pb.ops[0]   # the ladder R(abij) += Vv(abcd) T(cdij)
    orc = oracle_objects(pb)
    tags = dict(TAGS)
    dense = {n: O.dense_masked(orc[n], S.dense(orc[n].shape, 3, tags[n])) for n in (a, b, c)}
    packed = {n: O.pack(orc[n], dense[n]) for n in (a, b, c)}

    def body(rank, ctx):
        P = product_objects(tt, ctx, pb)
        if ctx.nranks > 1:
            tt.partition_split(ctx, P[c], cl, P[a], al, P[b], bl, group_dims=(0, 1))
            _mirror_rows(tt, P[c], P[a])
        bufs = {}
        for n in (a, b, c):   # device buffers start as NaN: only the uploads and the gather fill them
            bufs[n] = torch.full((P[n].storage_elems,), float("nan"), dtype=torch.float64, device="cuda")
            P[n].bind(bufs[n])
        host = {n: torch.from_numpy(packed[n].copy()).pin_memory() for n in (a, b, c)}
        ctx.set_profiling(True)
        tt.contract_host(ctx, P[c], cl, 1.0, 0.5, P[a], al, P[b], bl, host[a], host[b], host[c],
                         c_in=True, c_out=True)
        ctx.sync()
        launches = ctx.profile("tt_contract_dmma")[1]
        ctx.set_profiling(False)
        return P[c], host[c].numpy().copy(), launches

    one = run_ranks(tt, torch, 1, body)
    R1, seen1 = assemble([one[0][0]], [one[0][1]], one[0][0].packed_elems)
    res = run_ranks(tt, torch, p, body)
    Rp, seenp = assemble([r[0] for r in res], [r[1] for r in res], res[0][0].packed_elems)
    assert np.array_equal(seenp, seen1) and not np.isnan(Rp[seenp]).any()
    assert np.array_equal(Rp[seenp], R1[seen1]), "pipelined host contraction depends on the rank count"
    assert all(r[2] > 1 for r in res), [r[2] for r in res]   # chunked: one launch per chunk
    ref = O.pack(orc[c], O.contract(dense[c], cl, dense[a], al, dense[b], bl, 0.5, 1.0, cmask=O.nz_mask(orc[c])))
    err = np.abs(R1[seen1] - ref[seen1]).max() / np.abs(ref[seen1]).max()
    assert err <= 1e-11, err


@pytest.mark.parametrize("p", [2, 3])
def test_simulated_cholesky_owner_distributed_x(env, p):
    """The implicit Cholesky ladder with X owner-distributed (round robin; blocks held elsewhere NaN):
    each rank gathers X before building W; the assembled R2 equals bit for bit the run with X
    replicated and the 1-rank run."""
    tt, torch = env
    pb = _problem()

    def body_for(distributed):
        def body(rank, ctx):
            P = product_objects(tt, ctx, pb)
            so, sv = P["_keep"][1]["O"], P["_keep"][1]["V"]
            tL = tt.TiledIndexSpace(tt.IndexSpace(10), 5)
            X = tt.Tensor(ctx, [sv, sv, tL], spin=([0], [1]))
            if distributed:
                X.set_owner(np.where(X.nz > 0, np.arange(X.nblocks) % ctx.nranks, -1).astype(np.int32))
            else:
                X.set_owner(np.where(X.nz > 0, tt.TT_REPLICATED, -1).astype(np.int32))
            R2 = tt.Tensor(ctx, [sv, sv, so, so], spin=([0, 1], [2, 3]))
            tt.partition_split(ctx, R2, "abij", P["Vv"], "abcd", P["T"], "cdij", group_dims=(0, 1))
            xb = torch.empty(X.storage_elems, dtype=torch.float64, device="cuda")
            tb = torch.empty(P["T"].storage_elems, dtype=torch.float64, device="cuda")
            r2b = torch.full((R2.storage_elems,), float("nan"), dtype=torch.float64, device="cuda")
            X.bind(xb)
            P["T"].bind(tb)
            R2.bind(r2b)
            tt.fill_synthetic(ctx, X, 3, 9)
            tt.fill_synthetic(ctx, P["T"], 3, 5)
            tt.fill_synthetic(ctx, R2, 3, 10)
            if distributed:   # poison what this rank does not hold
                for blk in range(X.nblocks):
                    if X.nz[blk] and X.owner[blk] != rank:
                        o = int(X.storage_off[blk])
                        n = int(np.prod([int(d.offsets[t + 1] - d.offsets[t])
                                         for d, t in zip(X.dims, np.unravel_index(blk, X.grid))]))
                        xb[o:o + n] = float("nan")
            ws = torch.empty(P["T"].packed_elems + 32 + 12 ** 4 * 16, dtype=torch.float64, device="cuda")
            tt.contract_cholesky(ctx, R2, "abij", 1.0, 0.5, X, "abcd", P["T"], "cdij", ws)
            out = (R2, R2.download())
            ctx.sync()
            return out
        return body

    def assembled(res):
        return assemble([r[0] for r in res], [r[1] for r in res], res[0][0].packed_elems)

    R1, seen1 = assembled(run_ranks(tt, torch, 1, body_for(False)))
    Rr, seenr = assembled(run_ranks(tt, torch, p, body_for(False)))
    Rd, seend = assembled(run_ranks(tt, torch, p, body_for(True)))
    assert np.array_equal(seend, seen1) and not np.isnan(Rd[seend]).any()
    assert np.array_equal(Rd[seend], Rr[seenr]) and np.array_equal(Rd[seend], R1[seen1])


def test_simulated_ranks_with_wave_tail(env):
    """Row-split R on 3 simulated ranks with the wave tail forced on every contraction plan
    (TT_TAIL_SLOTS=2, warp-specialised variant forced): the owned R ranges equal bit for bit the 1-rank
    result without the tail."""
    import os
    tt, torch = env
    R1, seen1, _, _, _ = _run(tt, torch, 1, True)
    pb = _problem()
    os.environ["TT_TAIL_SLOTS"] = "2"
    os.environ["TT_FORCE_VARIANT"] = "3"
    try:
        res = run_ranks(tt, torch, 3, _body(tt, torch, pb, True))
    finally:
        os.environ.pop("TT_TAIL_SLOTS", None)
        os.environ.pop("TT_FORCE_VARIANT", None)
    Rp, seenp = assemble([r["R"][0] for r in res], [r["R"][1] for r in res], res[0]["R"][0].packed_elems)
    assert np.array_equal(seenp, seen1) and not np.isnan(Rp[seenp]).any()
    assert np.array_equal(Rp[seenp], R1[seen1])
