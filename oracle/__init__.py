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
                 and dense global arrays using the oracle's own addressing, sampled elements,
                 the unfactorized three-operand loop of Eq. cc9 (``contract3_naive``), slices (P159),
                 the Cholesky-factored operand of Eq. cc12 and the Freivalds check.
* ``layout.contract3_plan`` -- the cc9 pairings and their costs (reading R26); ``layout.tile_sub`` /
                 ``tile_range`` -- sub-spaces (P152, reading R29).
* ``triples`` -- the (T) energy of Eqs. cc14 / tensort / tensort2 (element loops and a by-triple form).
* ``ccsd``, ``sched`` -- the CCSD-shaped term list transcription and the scheduler levelization.

Pins (tests/test_oracle_pins.py, ``-m "not gpu"``): numpy.einsum (independent library routine)
on tiny shapes, integer-valued exactness, linearity, label-permutation equivalence, Kronecker and
rank-1 closed forms, the paper's Fig. 2 shapes (P125-140) and Fig. 5 program (P194-198 -> -10.0,
reading R2), SPEC worked examples (S55-87, S191, S200-202, S480-492), closed-form task counts
and FLOP fractions, antisymmetry (S633), zeros-in/zeros-out (S216); NEXT-3 pins
in tests/test_next3.py (pure-Python brute force, integer exactness of cc10/cc11 vs cc9, rank-1 closed
form, the n_o^4 n_u^4 / n_o^4 n_u^2 cost classes, Fig. 2 sub-spaces, slice additivity); (T) pins in
tests/test_triples.py (second-quantization evaluation of <Phi_ijk^abc|V_N T|Phi>, energy laws).
Every function is pinned; there is no "parity unpinned" entry.
"""
from . import layout, ops, triples  # noqa: F401
