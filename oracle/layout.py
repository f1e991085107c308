"""Oracle metadata: tilings, block maps, packed layout, task list, owner partition.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain Python loops, written from the paper:

* IndexSpace / TiledIndexSpace -- PAPER §3.1 P111, P116-127 (Fig. 2): an index range, tiled either
  with a fixed size (``tN{N,10}``, remainder in the last tile, reading R5) or custom sizes with full
  coverage (``tM{M,{10,20}}``).  Spin ranges (P138) split the tiling: a tile never straddles a spin
  boundary (S39, reading R6).
* Tensor blocks -- "indexed by the Cartesian product of the number of tiles on each dimension"
  (P111, P140), row-major block grid, row-major elements within a block (reading R9).
* Non-zero block map -- explicit, or the spin rule sum(spin of upper dims) == sum(spin of lower dims)
  over a per-tensor (upper, lower) position split (P138, reading R7).
* Packed storage -- only non-zero blocks are allocated (P210, third scheme); row-major block order,
  each block start rounded up to a multiple of 2 doubles (16 B) (reading R10).
* Default owners -- "allocates the tensor blocks in a round-robin fashion while taking block
  sparsity into account" (P210): owner = (ordinal among non-zero blocks) mod nranks.
* Task list -- for each non-zero C block (row-major), each contracted-tile tuple (row-major,
  contracted labels in order of first appearance in A): a task iff the A and B blocks are both
  non-zero (P111, P138, P210, P543; readings R8, R11).  Brute force over the full grid.
* LPT owner partition (reading R24): C blocks sorted by (cost desc, block id asc), each to the
  least-loaded rank, ties to the lowest rank.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from itertools import product
from typing import List, Optional, Sequence, Tuple


class OracleError(ValueError):
    pass


@dataclass
class IndexSpace:
    """P116-122: ``IndexSpace N{range(100)}``; ``ranges`` = [(begin, end, spin)] covering [0, extent)."""
    extent: int
    ranges: List[Tuple[int, int, int]] = field(default_factory=list)

    def __post_init__(self):
        if self.extent < 0:
            raise OracleError("negative extent")
        if self.ranges:
            pos = 0
            for b, e, s in self.ranges:
                if b != pos or e <= b:
                    raise OracleError("ranges must be ascending, non-empty and cover the space")
                pos = e
            if pos != self.extent:
                raise OracleError("ranges must cover the space")

    def segments(self):
        if self.ranges:
            return list(self.ranges)
        return [(0, self.extent, 0)] if self.extent > 0 else []


@dataclass
class TiledIndexSpace:
    space: IndexSpace
    offsets: List[int]        # ntiles + 1 split points
    tile_spin: List[int]      # spin of each tile (0 = no spin)

    @property
    def ntiles(self) -> int:
        return len(self.offsets) - 1

    def size(self, t: int) -> int:
        return self.offsets[t + 1] - self.offsets[t]


def tile_fixed(space: IndexSpace, tile: int) -> TiledIndexSpace:
    """P125 ``TiledIndexSpace tN{N, 10}``; remainder in the last tile of each spin range (R5, R6)."""
    if tile < 1:
        raise OracleError("tile < 1")
    offs, spins = [0], []
    for b, e, s in space.segments():
        p = b
        while p < e:
            q = min(p + tile, e)
            offs.append(q)
            spins.append(s)
            p = q
    return TiledIndexSpace(space, offs, spins)


def tile_custom(space: IndexSpace, sizes: Sequence[int]) -> TiledIndexSpace:
    """P126 ``TiledIndexSpace tM{M, {10,20}}`` -- arbitrary sizes with full coverage (P127)."""
    if any(int(s) < 1 for s in sizes):
        raise OracleError("tile size < 1")
    if sum(sizes) != space.extent:
        raise OracleError("tile sizes do not cover the index space")
    offs = [0]
    for s in sizes:
        offs.append(offs[-1] + int(s))
    spins = []
    segs = space.segments()
    for t in range(len(sizes)):
        lo, hi = offs[t], offs[t + 1]
        owner = [s for (b, e, s) in segs if b <= lo and hi <= e]
        if not owner:
            raise OracleError("tile straddles a spin range")
        spins.append(owner[0])
    return TiledIndexSpace(space, offs, spins)


def tile_sub(tis: TiledIndexSpace, begin: int, end: int) -> TiledIndexSpace:
    """P152/P159 sub-space ``tK("first")``: the tiles of ``tis`` covering [begin, end), which must start
    and end on tile boundaries; offsets relative to ``begin``."""
    if begin >= end or begin not in tis.offsets or end not in tis.offsets:
        raise OracleError("sub-space does not start and end on tile boundaries")
    t0, t1 = tis.offsets.index(begin), tis.offsets.index(end)
    sub = IndexSpace(end - begin)
    return TiledIndexSpace(sub, [o - begin for o in tis.offsets[t0:t1 + 1]], list(tis.tile_spin[t0:t1]))


def tile_range(tis: TiledIndexSpace, r: int) -> TiledIndexSpace:
    """P120-121 named range ("first" = range 0, "second" = range 1) of the tiled space's index space."""
    b, e, _ = tis.space.segments()[r]
    return tile_sub(tis, b, e)


@dataclass
class Tensor:
    dims: List[TiledIndexSpace]
    nz: List[int]                 # row-major over the block grid, 0/1
    nranks: int = 1

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def grid(self) -> Tuple[int, ...]:
        return tuple(d.ntiles for d in self.dims)

    @property
    def shape(self) -> Tuple[int, ...]:
        return tuple(d.space.extent for d in self.dims)

    def nblocks(self) -> int:
        n = 1
        for g in self.grid:
            n *= g
        return n

    def block_coords(self, bid: int) -> Tuple[int, ...]:
        """Row-major block id -> tile indices (P111: Cartesian product of tiles)."""
        c = []
        for g in reversed(self.grid):
            c.append(bid % g)
            bid //= g
        return tuple(reversed(c))

    def block_id(self, coords: Sequence[int]) -> int:
        b = 0
        for g, t in zip(self.grid, coords):
            b = b * g + t
        return b

    def block_extents(self, bid: int) -> Tuple[int, ...]:
        return tuple(d.size(t) for d, t in zip(self.dims, self.block_coords(bid)))

    def block_origin(self, bid: int) -> Tuple[int, ...]:
        return tuple(d.offsets[t] for d, t in zip(self.dims, self.block_coords(bid)))

    def block_volume(self, bid: int) -> int:
        v = 1
        for e in self.block_extents(bid):
            v *= e
        return v

    def blk_off(self) -> List[int]:
        """P210 (sparsity-aware scheme): packed offsets, -1 for zero blocks, 16-B aligned (R10)."""
        out, cur = [], 0
        for b in range(self.nblocks()):
            if self.nz[b]:
                cur = (cur + 1) // 2 * 2
                out.append(cur)
                cur += self.block_volume(b)
            else:
                out.append(-1)
        return out

    def packed_elems(self) -> int:
        offs = self.blk_off()
        end = 0
        for b, o in enumerate(offs):
            if o >= 0:
                end = max(end, o + self.block_volume(b))
        return (end + 1) // 2 * 2

    def owners(self) -> List[int]:
        """P210 third scheme: round-robin over non-zero blocks; -1 for zero blocks."""
        out, k = [], 0
        for b in range(self.nblocks()):
            if self.nz[b]:
                out.append(k % self.nranks)
                k += 1
            else:
                out.append(-1)
        return out


def tensor_dense_map(dims: Sequence[TiledIndexSpace], nranks: int = 1) -> Tensor:
    n = 1
    for d in dims:
        n *= d.ntiles
    return Tensor(list(dims), [1] * n, nranks)


def tensor_explicit(dims: Sequence[TiledIndexSpace], nz: Sequence[int], nranks: int = 1) -> Tensor:
    t = tensor_dense_map(dims, nranks)
    if len(nz) != t.nblocks():
        raise OracleError("nz length != number of blocks")
    t.nz = [1 if int(v) else 0 for v in nz]
    return t


def tensor_spin(dims: Sequence[TiledIndexSpace], upper: Sequence[int], lower: Sequence[int],
                nranks: int = 1) -> Tensor:
    """P138 spin block sparsity, reading R7: block non-zero iff the spin sums of the tiles at the
    ``upper`` positions and at the ``lower`` positions are equal."""
    t = tensor_dense_map(dims, nranks)
    nz = []
    for b in range(t.nblocks()):
        c = t.block_coords(b)
        su = sum(t.dims[p].tile_spin[c[p]] for p in upper)
        sl = sum(t.dims[p].tile_spin[c[p]] for p in lower)
        nz.append(1 if su == sl else 0)
    t.nz = nz
    return t


# ----------------------------------------------------------------------------- labelled contraction

@dataclass
class ContractionLabels:
    free_c: List[str]      # C labels in C order
    con: List[str]         # contracted labels, order of first appearance in A
    in_a: List[bool]       # per C label: True if it comes from A


def analyse_labels(c_lbl: str, a_lbl: str, b_lbl: str) -> ContractionLabels:
    """P174 ``C(i,a) += alpha * A(i,l) * B(l,a)``: l is contracted (in A and B, not in C)."""
    for s in (c_lbl, a_lbl, b_lbl):
        if len(set(s)) != len(s):
            raise OracleError("repeated label")
    con = [x for x in a_lbl if x in b_lbl and x not in c_lbl]
    for x in c_lbl:
        if (x in a_lbl) == (x in b_lbl):
            raise OracleError("C label must appear in exactly one of A, B")
    for x in a_lbl:
        if x not in c_lbl and x not in b_lbl:
            raise OracleError("dangling label in A")
    for x in b_lbl:
        if x not in c_lbl and x not in a_lbl:
            raise OracleError("dangling label in B")
    return ContractionLabels(list(c_lbl), con, [x in a_lbl for x in c_lbl])


def task_list(C: Tensor, c_lbl: str, A: Tensor, a_lbl: str, B: Tensor, b_lbl: str):
    """Canonical task list by brute force (reading R11).

    Returns (cblocks, ptr, a_blk, b_blk, cost): ``cblocks`` the non-zero C block ids in row-major
    order, CSR ``ptr`` over them, the A and B block ids of every task, and the FLOP cost
    2*prod(extents of all labels) summed per C block (S484-492: 2mnk per block GEMM)."""
    L = analyse_labels(c_lbl, a_lbl, b_lbl)
    tis = {}
    for T, lbl in ((C, c_lbl), (A, a_lbl), (B, b_lbl)):
        for d, x in zip(T.dims, lbl):
            tis.setdefault(x, d)
    con_grid = [tis[x].ntiles for x in L.con]
    cblocks, ptr, ab, bb, cost = [], [0], [], [], []
    for cb in range(C.nblocks()):
        ccoord = C.block_coords(cb)
        tile = dict(zip(c_lbl, ccoord))
        total = 0
        if not C.nz[cb]:
            continue
        for kt in product(*[range(n) for n in con_grid]):
            tile.update(zip(L.con, kt))
            a_id = A.block_id([tile[x] for x in a_lbl])
            b_id = B.block_id([tile[x] for x in b_lbl])
            if A.nz[a_id] and B.nz[b_id]:
                ab.append(a_id)
                bb.append(b_id)
                f = 2
                for x in list(c_lbl) + L.con:
                    f *= tis[x].size(tile[x])
                total += f
        cblocks.append(cb)
        ptr.append(len(ab))
        cost.append(total)
    return cblocks, ptr, ab, bb, cost


def lpt_partition(cost: Sequence[int], cblocks: Sequence[int], nranks: int) -> List[int]:
    """Deterministic LPT: order by (cost desc, block id asc); least-loaded rank, ties lowest rank."""
    order = sorted(range(len(cost)), key=lambda i: (-cost[i], cblocks[i]))
    load = [0] * nranks
    owner = [0] * len(cost)
    for i in order:
        r = min(range(nranks), key=lambda q: (load[q], q))
        owner[i] = r
        load[r] += cost[i]
    return owner


def lpt_partition_grouped(C: Tensor, cost: Sequence[int], cblocks: Sequence[int], group_dims: Sequence[int],
                          nranks: int) -> List[int]:
    """LPT over units of C blocks sharing the tile coordinates of ``group_dims`` (R24); unit cost =
    sum of its blocks' costs, unit id = its smallest block id.  Returns the owner of each C block."""
    units, ucost, uid, unit_of = {}, [], [], []
    for c, b in zip(cost, cblocks):
        key = tuple(C.block_coords(b)[d] for d in group_dims) if group_dims else (b,)
        if key not in units:
            units[key] = len(ucost)
            ucost.append(0)
            uid.append(b)
        ucost[units[key]] += c
        unit_of.append(units[key])
    uown = lpt_partition(ucost, uid, nranks)
    return [uown[u] for u in unit_of]


def partition_split(C: Tensor, cost: Sequence[int], cblocks: Sequence[int], group_dims: Sequence[int],
                    nranks: int):
    """Balanced partition with row splitting (reading R24b, SURVEY 8(e) "block splitting").

    Units (single blocks, or blocks sharing the tile coordinates of ``group_dims``, which then
    include dim 0) are ordered by (cost desc, smallest block id asc) and laid end to end on a cost
    axis of length W; rank r owns [floor(r*W/P), floor((r+1)*W/P)).  A unit that straddles a
    boundary is cut at the nearest row of its dim-0 tile: row = round_half_up((B_r - c0)*rows/cost).
    Returns {block: [(lo, hi, owner), ...]} for every non-zero C block in ``cblocks``."""
    units, order_keys = {}, []
    for c, b in zip(cost, cblocks):
        coords = C.block_coords(b)
        key = tuple(coords[d] for d in group_dims) if group_dims else (b,)
        if key not in units:
            units[key] = {"cost": 0, "id": b, "rows": C.dims[0].size(coords[0]), "blocks": []}
            order_keys.append(key)
        units[key]["cost"] += c
        units[key]["blocks"].append(b)
    order = sorted(order_keys, key=lambda k: (-units[k]["cost"], units[k]["id"]))
    W = sum(units[k]["cost"] for k in order)
    Bd = [r * W // nranks for r in range(nranks + 1)]
    out, cum = {}, 0
    for k in order:
        u = units[k]
        c0, c1, rows = cum, cum + u["cost"], u["rows"]
        cum = c1
        r0 = max([r for r in range(nranks) if Bd[r] <= c0] or [0])
        parts, cur, start = [], r0, 0
        if u["cost"] > 0:
            for r in range(r0 + 1, nranks):
                if Bd[r] >= c1:
                    break
                row = ((Bd[r] - c0) * rows * 2 + u["cost"]) // (2 * u["cost"])
                row = min(max(row, 0), rows)
                if row > start:
                    parts.append((start, row, cur))
                    start = row
                cur = r
        if rows > start:
            parts.append((start, rows, cur))
        for b in u["blocks"]:
            out[b] = parts
    return out


def cholesky_ladder_cost(C: Tensor, c_lbl: str, X: Tensor, v_lbl: str, B: Tensor, b_lbl: str):
    """Executed cost per non-zero C block of the implicit-operand ladder C += V(p,q,r,s) B (Eq. cc12,
    P312-318): the FLOPs of the block's tasks against the Coulomb operand
    W(p,q,r,s) = sum_L X(p,r,L) X(q,s,L), whose block (p_t,q_t,r_t,s_t) is non-zero iff X holds a
    non-zero block at (p_t,r_t,.) and at (q_t,s_t,.) (reading R19b), plus the formation of W's
    (p_t,q_t) row -- 2 N_L |p_t||q_t| sum over its non-zero (r_t,s_t) of |r_t||s_t| -- split evenly
    (floor) over the row's non-zero C blocks.  Returns (cblocks, cost) in task_list order."""
    p, q, r, s = v_lbl
    dims = {x: d for T, lbl in ((C, c_lbl), (B, b_lbl)) for x, d in zip(lbl, T.dims)}
    xpair = set()
    for xb in range(X.nblocks()):
        if X.nz[xb]:
            co = X.block_coords(xb)
            xpair.add((co[0], co[1]))
    vd = [dims[p], dims[q], dims[r], dims[s]]
    wnz = [1 if ((a, c) in xpair and (b, d) in xpair) else 0
           for a in range(vd[0].ntiles) for b in range(vd[1].ntiles)
           for c in range(vd[2].ntiles) for d in range(vd[3].ntiles)]
    W = tensor_explicit(vd, wnz)
    cblocks, _, _, _, cost = task_list(C, c_lbl, W, v_lbl, B, b_lbl)
    NL = X.dims[2].space.extent
    rows = {}
    for cb in cblocks:
        co = C.block_coords(cb)
        key = (co[c_lbl.index(p)], co[c_lbl.index(q)])
        rows[key] = rows.get(key, 0) + 1
    out = []
    for cb, c in zip(cblocks, cost):
        co = C.block_coords(cb)
        a, b = co[c_lbl.index(p)], co[c_lbl.index(q)]
        w = sum(vd[2].size(c2) * vd[3].size(d2) for c2 in range(vd[2].ntiles) for d2 in range(vd[3].ntiles)
                if (a, c2) in xpair and (b, d2) in xpair)
        build = 2 * NL * vd[0].size(a) * vd[1].size(b) * w
        out.append(c + build // rows[(a, b)])
    return cblocks, out


# ----------------------------------------------------------------------------- NEXT-3 factorization

def contract3_plan(C: Tensor, c_lbl: str, A: Tensor, a_lbl: str, B: Tensor, b_lbl: str, D: Tensor, d_lbl: str):
    """PAPER Eqs. cc9-cc11 (P293-311), reading R26: the three pairings (A*B)*D, (A*D)*B, (B*D)*A of the
    three-operand term, each as two binary contractions through an intermediate I whose labels are those
    of the pair (first operand's order, then the second's) that appear in the third operand or in C, and
    whose non-zero blocks are those receiving at least one task.  Cost = the FLOPs of both task lists;
    the cheapest pairing wins (ties: the first).  ``naive_macs`` = one product per combination of all
    label values with C, A, B, D blocks all non-zero (the unfactorized cc9 loop, brute force)."""
    ops = [(A, a_lbl), (B, b_lbl), (D, d_lbl)]
    flops, cand = [], []
    for x, y, z in ((0, 1, 2), (0, 2, 1), (1, 2, 0)):
        (X, xl), (Y, yl), (Z, zl) = ops[x], ops[y], ops[z]
        il, idims = "", []
        for T, l in ((X, xl), (Y, yl)):
            for d, ch in zip(T.dims, l):
                if (ch in zl or ch in c_lbl) and ch not in il:
                    il += ch
                    idims.append(d)
        if not il or len(il) > 8:
            flops.append(-1.0)
            cand.append(None)
            continue
        I = tensor_dense_map(idims)
        cbl, ptr, _, _, cost1 = task_list(I, il, X, xl, Y, yl)
        inz = [0] * I.nblocks()
        for g, cb in enumerate(cbl):
            if ptr[g + 1] > ptr[g]:
                inz[cb] = 1
        I.nz = inz
        _, _, _, _, cost2 = task_list(C, c_lbl, I, il, Z, zl)
        flops.append(float(sum(cost1) + sum(cost2)))
        cand.append(il)
    best = min((p for p in range(3) if flops[p] >= 0), key=lambda p: (flops[p], p))
    # naive loop count
    tis, order = {}, []
    for T, l in ((C, c_lbl), (A, a_lbl), (B, b_lbl), (D, d_lbl)):
        for d, ch in zip(T.dims, l):
            if ch not in tis:
                tis[ch] = d
                order.append(ch)
    macs = 0
    for tup in product(*[range(tis[ch].ntiles) for ch in order]):
        tile = dict(zip(order, tup))
        if all(T.nz[T.block_id([tile[ch] for ch in l])] for T, l in ((C, c_lbl), (A, a_lbl), (B, b_lbl),
                                                                      (D, d_lbl))):
            v = 1
            for ch in order:
                v *= tis[ch].size(tile[ch])
            macs += v
    return {"pair": best, "i_lbl": cand[best], "flops": flops, "naive_macs": float(macs)}
