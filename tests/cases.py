"""Test helper: one problem spec -> matching oracle objects and libtt objects.

The spec holds only sizes and maps (the paper's workload recipes); the oracle side and
the product side each build their own metadata from it."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

import synthetic as S
from oracle import layout as L
from oracle import ops as O

TAGS = {"A": 1, "B": 2, "C": 3}


@dataclass
class SpaceSpec:
    extent: int
    tile: Optional[int] = None
    sizes: Optional[Sequence[int]] = None
    spin_split: bool = False          # first half alpha, second half beta (reading R6)

    def ranges(self):
        if not self.spin_split:
            return None, None
        h = self.extent // 2
        return [(0, h), (h, self.extent)], [1, -1]


@dataclass
class TensorSpec:
    labels: str
    rule: Optional[Tuple] = None      # None = dense, ("spin", up, lo), ("nz", array)


@dataclass
class Problem:
    spaces: Dict[str, SpaceSpec]
    label_space: Dict[str, str]
    tensors: Dict[str, TensorSpec]
    ops: List[Tuple] = field(default_factory=list)


def oracle_objects(pb: Problem, nranks: int = 1):
    tis = {}
    for name, sp in pb.spaces.items():
        r, s = sp.ranges()
        space = L.IndexSpace(sp.extent, [(b, e, x) for (b, e), x in zip(r, s)] if r else [])
        tis[name] = L.tile_custom(space, sp.sizes) if sp.sizes is not None else L.tile_fixed(space, sp.tile)
    out = {}
    for tn, ts in pb.tensors.items():
        dims = [tis[pb.label_space[x]] for x in ts.labels]
        if ts.rule is None:
            out[tn] = L.tensor_dense_map(dims, nranks)
        elif ts.rule[0] == "spin":
            out[tn] = L.tensor_spin(dims, ts.rule[1], ts.rule[2], nranks)
        else:
            out[tn] = L.tensor_explicit(dims, list(ts.rule[1]), nranks)
    return out


def product_objects(tt, ctx, pb: Problem):
    keep = []
    tis = {}
    for name, sp in pb.spaces.items():
        r, s = sp.ranges()
        space = tt.IndexSpace(sp.extent, r, s)
        keep.append(space)
        tis[name] = tt.TiledIndexSpace(space, tile=sp.tile) if sp.sizes is None else tt.TiledIndexSpace(space, sizes=sp.sizes)
    out = {}
    for tn, ts in pb.tensors.items():
        dims = [tis[pb.label_space[x]] for x in ts.labels]
        if ts.rule is None:
            out[tn] = tt.Tensor(ctx, dims)
        elif ts.rule[0] == "spin":
            out[tn] = tt.Tensor(ctx, dims, spin=(ts.rule[1], ts.rule[2]))
        else:
            out[tn] = tt.Tensor(ctx, dims, nz=np.asarray(ts.rule[1], dtype=np.uint8))
    out["_keep"] = (keep, tis)
    return out


def ccsd_problem(O_: int, V_: int, tO: int, tV: int, spin: bool, terms=("ladder", "ring", "hh")) -> Problem:
    """Synthetic CC maps of reading R7: R{ab|ij}, V{ab|cd}, T{cd|ij}, ring A{ac|ik}, B{kb|cj}, W{kl|ij}."""
    spaces = {"O": SpaceSpec(O_, tile=tO, spin_split=spin), "V": SpaceSpec(V_, tile=tV, spin_split=spin)}
    ls = {x: "V" for x in "abcdef"}
    ls.update({x: "O" for x in "ijklmn"})
    sp = (lambda up, lo: ("spin", up, lo)) if spin else (lambda up, lo: None)
    tensors = {"R": TensorSpec("abij", sp([0, 1], [2, 3]))}
    ops = []
    if "ladder" in terms:
        tensors["Vv"] = TensorSpec("abcd", sp([0, 1], [2, 3]))
        tensors["T"] = TensorSpec("cdij", sp([0, 1], [2, 3]))
        ops.append(("R", "abij", "Vv", "abcd", "T", "cdij"))
    if "ring" in terms:
        tensors["Ta"] = TensorSpec("acik", sp([0, 1], [2, 3]))
        tensors["Wr"] = TensorSpec("cbkj", sp([2, 1], [0, 3]))
        ops.append(("R", "abij", "Ta", "acik", "Wr", "cbkj"))
    if "hh" in terms:
        tensors["Tb"] = TensorSpec("abkl", sp([0, 1], [2, 3]))
        tensors["Wh"] = TensorSpec("klij", sp([0, 1], [2, 3]))
        ops.append(("R", "abij", "Tb", "abkl", "Wh", "klij"))
    return Problem(spaces, ls, tensors, ops)


def host_packed(T: L.Tensor, seed: int, tag: int, kind: int = S.KIND_UNIFORM) -> np.ndarray:
    """Packed storage filled with generator values at global indices (zero blocks absent)."""
    D = S.dense(T.shape, seed, tag, kind)
    return O.pack(T, D)
