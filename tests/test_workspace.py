"""The caller-provided device workspace (include/tt.h tt_workspace_*; P182-186: the
ExecutionContext carries the memory manager).

CPU: the calls are exported and behave on a host-only context.  GPU: a context without a workspace
refuses device work (TT_E_WORKSPACE) and reports what it needs; a workspace far smaller than the
workload's metadata forces least-recently-used plan eviction and the results stay bitwise equal to a
roomy workspace; re-binding drops plans and device metadata and the next calls rebuild them; a captured
scheduler graph pins its plans (eviction never frees them) and forbids re-binding."""
import ctypes

import numpy as np
import pytest

import synthetic as S
from oracle import ops as O
from tests.cases import ccsd_problem, oracle_objects, product_objects


def test_host_ctx_workspace_calls():
    import paper_2201_01257_b200 as tt
    c = tt.Context(device=-1)
    assert c.workspace_bytes() == 1 << 20          # kWsMin before any call
    assert c.workspace_info() == {"bound": 0, "live": 0, "high": 0}
    c.set_plan_limit(3)
    c.clear_plans()
    with pytest.raises(tt.TTError) as e:
        c.set_plan_limit(0)
    assert e.value.name == "TT_E_ARG"
    with pytest.raises(tt.TTError) as e:           # host-only: no device to bind on
        tt._check(tt._lib.tt_workspace_bind(c.h, ctypes.c_void_p(256), 1 << 20))
    assert e.value.name == "TT_E_STATE"
    c.close()


# ----------------------------------------------------------------------------------------------- GPU

def _setup(tt, torch, ctx, pb, seed=1):
    orc = oracle_objects(pb)
    P = product_objects(tt, ctx, pb)
    keep, dense = [], {}
    for i, name in enumerate(sorted(orc)):
        D = O.dense_masked(orc[name], S.dense(orc[name].shape, seed, 1 + i))
        dense[name] = D
        buf = torch.from_numpy(O.pack(orc[name], D)).cuda()
        P[name].bind(buf)
        keep.append(buf)
    return orc, P, keep, dense


def _run_all(tt, ctx, pb, P, reps=2):
    for _ in range(reps):
        for (c, cl, a, al, b, bl) in pb.ops:
            tt.contract(ctx, P[c], cl, 1.0, 0.5, P[a], al, P[b], bl)
    return {c: P[c].download() for (c, *_r) in pb.ops}


@pytest.mark.gpu
def test_no_workspace_is_refused_then_bind_works():
    import torch
    import paper_2201_01257_b200 as tt
    torch.cuda.init()
    h = ctypes.c_void_p()
    tt._check(tt._lib.tt_ctx_create(0, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), 0, 1, None,
                                    ctypes.byref(h)))
    raw = tt.Context.__new__(tt.Context)
    raw.h, raw.device, raw.rank, raw.nranks, raw.sim, raw._ws = h, 0, 0, 1, None, None
    pb = ccsd_problem(4, 8, 4, 4, False, terms=("ladder",))
    orc, P, keep, dense = _setup(tt, torch, raw, pb)
    c, cl, a, al, b, bl = pb.ops[0]
    with pytest.raises(tt.TTError) as e:
        tt.contract(raw, P[c], cl, 1.0, 1.0, P[a], al, P[b], bl)
    assert e.value.name == "TT_E_WORKSPACE"
    with pytest.raises(tt.TTError) as e:
        tt.set_(raw, P[c], 1.0)
    assert e.value.name == "TT_E_WORKSPACE"
    assert raw.workspace_bytes() >= 1 << 20
    raw.bind_workspace(raw.workspace_bytes())
    tt.contract(raw, P[c], cl, 1.0, 1.0, P[a], al, P[b], bl)
    got = P[c].download()
    raw.sync()
    ref = O.pack(orc[c], O.contract(dense[c], cl, dense[a], al, dense[b], bl, 1.0, 1.0, cmask=O.nz_mask(orc[c])))
    assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max()
    info = raw.workspace_info()
    assert 0 < info["live"] <= info["high"] <= info["bound"]
    raw.close()


@pytest.mark.gpu
def test_small_workspace_evicts_and_matches():
    """Three CCSD-shaped terms whose plans do not fit together in the small workspace: every call
    evicts the others' plans (LRU, after a device drain) and rebuilds its own; the results are bitwise
    those of a roomy workspace (R12: the kernels' summation order does not depend on the plan's address)."""
    import torch
    import paper_2201_01257_b200 as tt
    torch.cuda.init()
    st = torch.cuda.current_stream().cuda_stream
    pb = ccsd_problem(12, 24, 3, 4, True)
    big = tt.Context(device=0, stream=st)
    _, Pb, kb, _ = _setup(tt, torch, big, pb)
    ref = _run_all(tt, big, pb, Pb)
    big.sync()
    need = big.workspace_info()["high"]
    big.close()
    small = tt.Context(device=0, stream=st, workspace_bytes=need * 6 // 10)   # holds the largest plan, not all
    _, Ps, ks, _ = _setup(tt, torch, small, pb)
    got = _run_all(tt, small, pb, Ps)
    small.sync()
    for k in ref:
        assert np.array_equal(ref[k], got[k]), k
    info = small.workspace_info()
    assert info["high"] <= info["bound"] < need
    # plan limit 1: every call replaces the previous plan in the cache
    small.set_plan_limit(1)
    _, Ps2, ks2, _ = _setup(tt, torch, small, pb)
    got2 = _run_all(tt, small, pb, Ps2)
    small.sync()
    for k in ref:
        assert np.array_equal(ref[k], got2[k]), k
    # a workspace too small for even one plan: TT_E_WORKSPACE, and tt_workspace_bytes says how much
    tiny = tt.Context(device=0, stream=st, workspace_bytes=4096)
    _, Pt, kt, _ = _setup(tt, torch, tiny, pb)
    c, cl, a, al, b, bl = pb.ops[0]
    with pytest.raises(tt.TTError) as e:
        tt.contract(tiny, Pt[c], cl, 1.0, 0.5, Pt[a], al, Pt[b], bl)
    assert e.value.name == "TT_E_WORKSPACE"
    for attempt in range(12):   # grow to what the failed calls reported (each failure names its need)
        tiny.bind_workspace(max(tiny.workspace_bytes(), 2 * tiny.workspace_info()["bound"]))
        try:
            tt.contract(tiny, Pt[c], cl, 1.0, 0.0, Pt[a], al, Pt[b], bl)   # alpha 0: R unchanged
            for (c2, cl2, a2, al2, b2, bl2) in pb.ops[1:]:
                tt.contract(tiny, Pt[c2], cl2, 1.0, 0.0, Pt[a2], al2, Pt[b2], bl2)
            break
        except tt.TTError as e2:
            assert e2.name == "TT_E_WORKSPACE"
    got3 = _run_all(tt, tiny, pb, Pt)
    tiny.sync()
    for k in ref:
        assert np.array_equal(ref[k], got3[k]), k
    small.close()
    tiny.close()


@pytest.mark.gpu
def test_rebind_rebuilds_and_graph_pins_plans():
    import torch
    import paper_2201_01257_b200 as tt
    torch.cuda.init()
    st = torch.cuda.current_stream().cuda_stream
    pb = ccsd_problem(8, 16, 2, 4, True)
    ctx = tt.Context(device=0, stream=st)
    _, P, keep, _ = _setup(tt, torch, ctx, pb)
    ref = _run_all(tt, ctx, pb, P, reps=1)
    ctx.sync()
    # re-bind: plans and tensor metadata are dropped and rebuilt on the next calls
    _, P1, keep1, _ = _setup(tt, torch, ctx, pb)
    ctx.bind_workspace(8 << 20)
    got = _run_all(tt, ctx, pb, P1, reps=1)
    ctx.sync()
    for k in ref:
        assert np.array_equal(ref[k], got[k]), k
    # a captured graph holds its plans: clearing the cache / evicting cannot free them, and re-binding
    # is refused while it lives
    _, P2, keep2, _ = _setup(tt, torch, ctx, pb)
    s = tt.Scheduler(ctx)
    for (c, cl, a, al, b, bl) in pb.ops:
        s.contract(P2[c], cl, 1.0, 0.5, P2[a], al, P2[b], bl)
    s.capture()
    ctx.clear_plans()
    ctx.set_plan_limit(1)
    _, P3, keep3, _ = _setup(tt, torch, ctx, ccsd_problem(6, 14, 3, 5, True))   # other plans churn the cache
    for (c, cl, a, al, b, bl) in ccsd_problem(6, 14, 3, 5, True).ops:
        tt.contract(ctx, P3[c], cl, 0.0, 1.0, P3[a], al, P3[b], bl)
    with pytest.raises(tt.TTError) as e:
        ctx.bind_workspace(16 << 20)
    assert e.value.name == "TT_E_STATE"
    s.replay()
    ctx.sync()
    for (c, *_r) in pb.ops:
        assert np.array_equal(ref[c], P2[c].download()), c
    s.close()
    ctx.bind_workspace(16 << 20)   # allowed again once the graph is gone
    ctx.close()
