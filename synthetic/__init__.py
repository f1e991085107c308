"""Seeded synthetic inputs shared by the oracle side and the test/bench harness.

This module holds NO arithmetic of the method (no tiling, no block maps, no contraction).
It defines only the counter-based value generator of SURVEY.md §8(d) "Inputs":

    value(seed, tag, g) = u01(splitmix64(seed ^ (tag * 0x9E3779B97F4A7C15) ^ g)) * 2 - 1      (uniform)
    value(seed, tag, g) = (splitmix64(...) mod 5) - 2                                          (integer)

where ``g`` is the GLOBAL row-major linear index of the element over the tensor's full (dense)
extents, and u01 keeps the top 53 bits (x >> 11) * 2^-53.  Because a value is a pure function of
the global index, any layout bug on either side changes values and cannot hide.

The CUDA library implements the same generator on the device (``tt_fill_synthetic``) so that the
bench can fill tensors of many GB without a host round trip; ``tests/test_gpu_parity.py`` checks
the device fill against this module bit for bit.  The oracle never sees device-generated data.

Tensor tags: A=1, B=2, C=3, V=4, T=5, W=6, X=7.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
TAGS = {"A": 1, "B": 2, "C": 3, "V": 4, "T": 5, "W": 6, "X": 7}
KIND_UNIFORM = 0
KIND_INTEGER = 1


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def key(seed: int, tag: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return np.uint64(seed) ^ (np.uint64(tag) * GOLDEN)


def values(seed: int, tag: int, gidx, kind: int = KIND_UNIFORM) -> np.ndarray:
    """Generator values at global linear indices ``gidx`` (any int array)."""
    g = np.asarray(gidx, dtype=np.int64).astype(np.uint64)
    h = splitmix64(key(seed, tag) ^ g)
    if kind == KIND_UNIFORM:
        return (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0) * 2.0 - 1.0
    if kind == KIND_INTEGER:
        return (h % np.uint64(5)).astype(np.int64).astype(np.float64) - 2.0
    raise ValueError(f"unknown kind {kind}")


def dense(shape, seed: int, tag: int, kind: int = KIND_UNIFORM) -> np.ndarray:
    """Full dense tensor of generator values (row-major global index)."""
    n = int(np.prod(shape, dtype=np.int64)) if len(shape) else 1
    return values(seed, tag, np.arange(n, dtype=np.int64), kind).reshape(shape)


def linear_index(shape, idx) -> np.ndarray:
    """Row-major linear index of index tuples ``idx`` (array [..., order]) in ``shape``."""
    idx = np.asarray(idx, dtype=np.int64)
    g = np.zeros(idx.shape[:-1], dtype=np.int64)
    for d, n in enumerate(shape):
        g = g * int(n) + idx[..., d]
    return g
