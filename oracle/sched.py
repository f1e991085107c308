"""Oracle of the scheduler's levelization -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

PAPER P215: operations that share a tensor where one of them updates it conflict and cannot run in
the same batch; batches ("levels") minimise the global synchronisations.  Reading R25 (after SPEC
S464-472): level(op) = 1 + max level over earlier conflicting ops, 0 if none.

Pins (tests/test_sched.py): Fig. 5 -> 3 levels (S470), and on random queues the number of levels
equals the longest chain of pairwise-conflicting ops in queue order found by brute force over all
subsequences (an independent computation), with no conflict inside a level."""
from itertools import combinations
from typing import List, Sequence, Set, Tuple

Op = Tuple[Set[str], Set[str]]   # (reads, writes)


def conflicts(x: Op, y: Op) -> bool:
    rx, wx = x
    ry, wy = y
    return bool(wx & (wy | ry)) or bool(wy & rx)


def levelize(ops: Sequence[Op]) -> List[int]:
    lv = []
    for i, op in enumerate(ops):
        lv.append(max([lv[j] + 1 for j in range(i) if conflicts(op, ops[j])] or [0]))
    return lv


def longest_chain_bruteforce(ops: Sequence[Op]) -> int:
    n = len(ops)
    best = 1 if n else 0
    for k in range(2, n + 1):
        for sub in combinations(range(n), k):
            if all(conflicts(ops[sub[t]], ops[sub[t + 1]]) for t in range(k - 1)):
                best = max(best, k)
    return best
