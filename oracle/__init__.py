"""CPU oracle for the tiled block-sparse FP64 contraction path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package ``paper_2201_01257_b200``
never imports it and shares no code with it (no kernels, headers, helpers or tables); the only
module both sides use is ``synthetic`` (seeded input values, no method arithmetic).

What it defines (each function cites the passage it follows; PAPER.md = /root/reference/PAPER.md
line numbers ``P<n>``, SPEC.md ``S<n>``, readings ``R<n>`` are listed in DESIGN.md §3):

* ``layout``  -- index spaces, tilings, block grids, non-zero block maps, packed offsets, owners,
                 the canonical task list (brute force) and the LPT owner partition.
* ``ops``     -- set / add / contraction / scalar contraction over dense global arrays
                 (plain nested loops in ``oracle.c``), pack/unpack between packed block storage
                 and dense global arrays using the oracle's own addressing, sampled elements.

Pins (tests/test_oracle_pins.py, ``-m "not gpu"``): numpy.einsum (independent library routine)
on tiny shapes, integer-valued exactness, linearity, label-permutation equivalence, Kronecker and
rank-1 closed forms, the paper's Fig. 2 shapes (P125-140) and Fig. 5 program (P194-198 -> -10.0,
reading R2), SPEC worked examples (S55-87, S191, S200-202, S480-492), closed-form task counts
and FLOP fractions, antisymmetry (S633), zeros-in/zeros-out (S216).
Every function is pinned; there is no "parity unpinned" entry.
"""
from . import layout, ops  # noqa: F401
