"""GPU parity of the element operations (SURVEY §8(a) A8 add, A10 scalar) under general label maps.

Blocks of one operation may need different kernel modes: a transposing map is a 32x32 shared-memory
transpose for most blocks, but a block whose remainder tile has extent 1 (S77: extent 7, tile 3 ->
{3, 3, 1}) degenerates to the generic decode.  Every block of such a plan must be computed (VERDICT r1
item 1).  Label maps: 2-, 3- and 4-cycles (P173 AddOp "with respect to the label permutation"), on
dense ragged tilings with extent-1 tails and on spin-split tilings (reading R6), beta in {0, 1, -0.5}."""
import numpy as np
import pytest

import synthetic as S
from oracle import ops as O
from tests.cases import Problem, SpaceSpec, TensorSpec, oracle_objects, product_objects

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2201_01257_b200 as tt
    torch.cuda.init()
    return tt, torch


def _spin_rule(lbl, up_labels):
    return ("spin", [lbl.index(x) for x in up_labels], [lbl.index(x) for x in lbl if x not in up_labels])


SPACES = {
    # dense, extent-1 remainder tiles ({3,3,1} of S77; 45 = 2*32 - 19 wide tiles of {32, 12, 1})
    "tail1": {"O": SpaceSpec(7, tile=3), "V": SpaceSpec(45, sizes=[32, 12, 1])},
    # spin halves with extent-1 tails per half ({3,3,1 | 3,3,1}; {20,3,1 | 20,3,1})
    "spin_tail1": {"O": SpaceSpec(14, sizes=[3, 3, 1, 3, 3, 1], spin_split=True),
                   "V": SpaceSpec(48, sizes=[20, 3, 1, 20, 3, 1], spin_split=True)},
    # ragged spin tiles wider than 32 (several transpose tiles per block and ragged tile edges)
    "spin_wide": {"O": SpaceSpec(18, tile=5, spin_split=True), "V": SpaceSpec(90, tile=37, spin_split=True)},
    # rows of 8..12 along j (rows / row-tile modes: aibj, biaj keep j innermost in both operands)
    "rows": {"O": SpaceSpec(40, tile=12, spin_split=True), "V": SpaceSpec(24, tile=7, spin_split=True)},
}
MAPS4 = ["bija", "jabi", "ijab", "baji", "abji", "ajbi", "jiba", "aibj", "biaj", "baij"]


def _run_add_scalar(tt, torch, spaces, c_lbl, a_lbl, spin):
    ls = {"a": "V", "b": "V", "c": "V", "i": "O", "j": "O"}
    if spin and len(c_lbl) == 4:
        c_rule, a_rule = _spin_rule(c_lbl, "ab"), _spin_rule(a_lbl, "ab")
    elif spin and len(c_lbl) == 2:
        c_rule, a_rule = _spin_rule(c_lbl, "a"), _spin_rule(a_lbl, "a")
    else:
        c_rule = a_rule = None
    pb = Problem(spaces, ls, {"C": TensorSpec(c_lbl, c_rule), "A": TensorSpec(a_lbl, a_rule)})
    ctx = tt.Context(device=0, stream=torch.cuda.current_stream().cuda_stream)
    orc = oracle_objects(pb)
    P = product_objects(tt, ctx, pb)
    dense = {n: O.dense_masked(orc[n], S.dense(orc[n].shape, 17, t)) for n, t in (("C", 3), ("A", 1))}
    bufs = {}
    for n in ("C", "A"):
        bufs[n] = torch.from_numpy(O.pack(orc[n], dense[n])).cuda()
        P[n].bind(bufs[n])
    mask = O.nz_mask(orc["C"])
    for beta in (1.0, 0.0, -0.5):
        tt.add(ctx, P["C"], c_lbl, beta, 0.75, P["A"], a_lbl)
        got = P["C"].download()
        ctx.sync()
        ref = O.add(dense["C"], c_lbl, dense["A"], a_lbl, 0.75, beta, cmask=mask)
        r = O.pack(orc["C"], ref)
        err = np.abs(got - r).max() / np.abs(r).max()
        assert err <= 1e-15, (c_lbl, a_lbl, beta, err)
        dense["C"] = ref
    for (x, xl, y, yl) in (("A", a_lbl, "C", c_lbl), ("C", c_lbl, "A", a_lbl)):
        s = tt.contract_scalar(ctx, -0.5, P[x], xl, P[y], yl)
        so = O.scalar(dense[x], xl, dense[y], yl, -0.5)
        assert abs(s - so) <= 1e-13 * max(abs(so), 1.0), (xl, yl, s, so)
    ctx.close()


@pytest.mark.parametrize("space", list(SPACES))
@pytest.mark.parametrize("a_lbl", MAPS4)
def test_add_scalar_4d_label_maps(env, space, a_lbl):
    tt, torch = env
    _run_add_scalar(tt, torch, SPACES[space], "abij", a_lbl, space.startswith("spin"))


@pytest.mark.parametrize("space", list(SPACES))
@pytest.mark.parametrize("c_lbl,a_lbl", [("abc", "cab"), ("abc", "bca"), ("ia", "ai"), ("ai", "ia")])
def test_add_scalar_3d_2d_label_maps(env, space, c_lbl, a_lbl):
    tt, torch = env
    spin = space.startswith("spin") and len(c_lbl) == 2
    _run_add_scalar(tt, torch, SPACES[space], c_lbl, a_lbl, spin)


def test_integer_add_bit_exact(env):
    """Integer-valued inputs: add is exact whatever the kernel mode."""
    tt, torch = env
    spaces = SPACES["tail1"]
    ls = {"a": "V", "b": "V", "i": "O", "j": "O"}
    pb = Problem(spaces, ls, {"C": TensorSpec("abij"), "A": TensorSpec("jabi")})
    ctx = tt.Context(device=0, stream=torch.cuda.current_stream().cuda_stream)
    orc = oracle_objects(pb)
    P = product_objects(tt, ctx, pb)
    dense = {n: S.dense(orc[n].shape, 5, t, S.KIND_INTEGER) for n, t in (("C", 3), ("A", 1))}
    bufs = {n: torch.from_numpy(O.pack(orc[n], dense[n])).cuda() for n in ("C", "A")}
    for n in ("C", "A"):
        P[n].bind(bufs[n])
    tt.add(ctx, P["C"], "abij", 2.0, -3.0, P["A"], "jabi")
    got = P["C"].download()
    ctx.sync()
    assert np.array_equal(got, O.pack(orc["C"], O.add(dense["C"], "abij", dense["A"], "jabi", -3.0, 2.0)))
    ctx.close()


@pytest.mark.gpu
def test_add_bits_independent_of_block_mode():
    """A permuted add gives the same bits whether a block runs as 32x32 transpose tiles (whole block) or as
    generic segments (row-split block): one rounding order, beta*x + alpha*y = fma(beta, x, alpha*y), in
    every element kernel (R12: results independent of the partition)."""
    import torch
    import paper_2201_01257_b200 as tt
    from tests.cases import ccsd_problem, oracle_objects, product_objects
    import synthetic as S
    from oracle import ops as O
    pb = ccsd_problem(12, 24, 6, 8, True, terms=("ladder",))
    orc = oracle_objects(pb)
    outs = []
    for split in (False, True):
        ctx = tt.Context(device=0, stream=torch.cuda.current_stream().cuda_stream)
        P = product_objects(tt, ctx, pb)
        R, T = P["R"], P["T"]
        if split:   # every non-zero R block owned by rank 0 in two row parts: segments instead of tiles
            parts = []
            for blk in range(R.nblocks):
                if R.nz[blk]:
                    e0 = int(np.diff(R.dims[0].offsets)[np.unravel_index(blk, R.grid)[0]])
                    parts += [(blk, 0, e0 // 2, 0), (blk, e0 // 2, e0, 0)]
            R.set_parts(parts)
        bR = torch.from_numpy(O.pack(orc["R"], O.dense_masked(orc["R"], S.dense(orc["R"].shape, 4, 3)))).cuda()
        bT = torch.from_numpy(O.pack(orc["T"], O.dense_masked(orc["T"], S.dense(orc["T"].shape, 4, 5)))).cuda()
        R.bind(bR)
        T.bind(bT)
        tt.add(ctx, R, "abij", 0.7, -1.3, T, "abji")
        outs.append(R.download())
        ctx.sync()
        ctx.close()
    assert np.array_equal(outs[0], outs[1])
