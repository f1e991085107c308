"""Test harness: run one SPMD body on p SIMULATED ranks of one GPU (tt_sim_create / tt_ctx_create_sim),
one host thread per rank, exactly as one process per GPU would run it."""
from __future__ import annotations

import threading

import numpy as np


def run_ranks(tt, torch, p: int, body, timeout: float = 600.0):
    """body(rank, ctx) -> result, called on p threads (own CUDA stream each); returns [result per rank].
    A rank that raises fails the run (the others may then block in a collective: the join times out)."""
    group = tt.SimGroup(0, p)
    streams = [torch.cuda.Stream(device=0) for _ in range(p)]
    ctxs = [tt.Context(stream=s.cuda_stream, rank=r, sim=group) for r, s in enumerate(streams)]
    out, errors = [None] * p, []

    def run(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(streams[r]):
                out[r] = body(r, ctxs[r])
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001
            errors.append((r, e))

    th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(p)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    if any(t.is_alive() for t in th):
        raise RuntimeError(f"simulated ranks did not finish within {timeout} s (errors: {errors})")
    if errors:
        raise errors[0][1]
    for c in ctxs:
        c.close()
    group.close()
    return out


def owned_ranges(T, rank):
    """[(global packed begin, end, storage begin)] of the element ranges of T that `rank` owns."""
    out = []
    for blk in range(T.nblocks):
        if not T.nz[blk]:
            continue
        o, so = int(T.blk_off[blk]), int(T.storage_off[blk])
        ext = [int(d.offsets[t + 1] - d.offsets[t]) for d, t in zip(T.dims, np.unravel_index(blk, T.grid))]
        n = int(np.prod(ext))
        if T.owner[blk] == rank:
            out.append((o, o + n, so))
        inner = n // ext[0]
        for (bb, lo, hi, ow) in T.parts:
            if bb == blk and ow == rank:
                out.append((o + lo * inner, o + hi * inner, so + lo * inner))
    return out


def assemble(T_of_rank, stor_of_rank, packed_elems):
    """Global packed array from every rank's owned ranges (each element owned by exactly one rank);
    elements nobody owns (padding) are NaN, elements owned twice raise."""
    g = np.full(packed_elems, np.nan)
    seen = np.zeros(packed_elems, dtype=bool)
    for r, (T, st) in enumerate(zip(T_of_rank, stor_of_rank)):
        for (b, e, s) in owned_ranges(T, r):
            assert not seen[b:e].any(), "element owned by two ranks"
            seen[b:e] = True
            g[b:e] = st[s:s + (e - b)]
    return g, seen
