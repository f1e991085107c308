"""World-size-2 (and 3) CPU test of the N > 1 host logic over torch.distributed gloo.

Each process builds the same SPMD metadata in a host-only libtt context (rank r of N): LPT owner
partition of the output blocks, default round-robin owners of the inputs, and its gather plan.  The
plan is then EXECUTED with gloo point-to-point messages on CPU buffers in which a rank initially
holds only its own blocks (NaN elsewhere).  Afterwards every input block read by the rank's tasks
must hold the generator values (no missing block, nothing received twice), and all ranks must
agree on partitions and plan symmetry."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, split):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2201_01257_b200 as tt
        import synthetic as S
        from oracle import layout as L
        from oracle import ops as O
        from tests.cases import ccsd_problem, oracle_objects, product_objects
        ctx = tt.Context(device=-1, rank=rank, nranks=world)
        pb = ccsd_problem(8, 12, 2, 3, True)
        orc = oracle_objects(pb)
        P = product_objects(tt, ctx, pb)
        results = []
        for (c, cl, a, al, b, bl) in pb.ops:
            if split:
                tt.partition_split(ctx, P[c], cl, P[a], al, P[b], bl)
            else:
                P[c].set_owner(tt.partition_lpt(ctx, P[c], cl, P[a], al, P[b], bl))
            mine_owner = (P[c].owner.tolist(), P[c].parts)
            owns = [None] * world
            dist.all_gather_object(owns, mine_owner)
            assert all(o == owns[0] for o in owns), "partition differs across ranks"
            recv, send = tt.gather_plan(ctx, P[c], cl, P[a], al, P[b], bl)
            # local buffers: generator values on held blocks, NaN elsewhere
            bufs = []
            for name, tag in ((a, 1), (b, 2)):
                full = O.pack(orc[name], S.dense(orc[name].shape, 5, tag))
                mine = np.full_like(full, np.nan)
                T = P[name]
                for blk in range(T.nblocks):
                    if T.nz[blk] and T.owner[blk] in (rank, tt.TT_REPLICATED):
                        o, n = T.blk_off[blk], orc[name].block_volume(blk)
                        mine[o:o + n] = full[o:o + n]
                    for (bb, lo, hi, ow) in T.parts:
                        if bb == blk and ow == rank:
                            inner = orc[name].block_volume(blk) // orc[name].block_extents(blk)[0]
                            o = T.blk_off[blk]
                            mine[o + lo * inner:o + hi * inner] = full[o + lo * inner:o + hi * inner]
                bufs.append((T, orc[name], full, mine))
            reqs = []
            for op, blk, peer, e0, e1 in send.tolist():
                T, ot, full, mine = bufs[op]
                o = T.blk_off[blk]
                assert not np.any(np.isnan(mine[o + e0:o + e1])), "sending data not held"
                reqs.append(dist.isend(torch.from_numpy(mine[o + e0:o + e1].copy()), dst=peer,
                                       tag=(op * 100003 + blk) * 64 + e0 % 64))
            incoming = []
            for op, blk, peer, e0, e1 in recv.tolist():
                T, ot, full, mine = bufs[op]
                t = torch.empty(e1 - e0, dtype=torch.float64)
                reqs.append(dist.irecv(t, src=peer, tag=(op * 100003 + blk) * 64 + e0 % 64))
                incoming.append((op, blk, e0, t))
            for r in reqs:
                r.wait()
            for op, blk, e0, t in incoming:
                T, ot, full, mine = bufs[op]
                o = T.blk_off[blk] + e0
                assert np.all(np.isnan(mine[o:o + t.numel()])), "received a range already held"
                mine[o:o + t.numel()] = t.numpy()
            # every block read by my tasks is now valid and correct
            cb, ptr, ab, bb, _ = L.task_list(orc[c], cl, orc[a], al, orc[b], bl)
            for g, cblk in enumerate(cb):
                rows = [(0, orc[c].block_extents(cblk)[0])] if P[c].owner[cblk] == rank else \
                    [(lo, hi) for (bb_, lo, hi, ow) in P[c].parts if bb_ == cblk and ow == rank]
                for (lo, hi) in rows:
                    for t in range(ptr[g], ptr[g + 1]):
                        for op, blk, lbl in ((0, ab[t], al), (1, bb[t], bl)):
                            T, ot, full, mine = bufs[op]
                            o, n = T.blk_off[blk], ot.block_volume(blk)
                            if lbl[0] == cl[0]:    # only the matching rows are needed
                                inner = n // ot.block_extents(blk)[0]
                                o, n = o + lo * inner, (hi - lo) * inner
                            assert np.array_equal(mine[o:o + n], full[o:o + n])
            results.append((len(recv), len(send)))
        q.put((rank, "ok", results))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("split", [False, True])
def test_gather_plan_executes_over_gloo(world, split):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, split)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, status, info in out:
        assert status == "ok", info
    # something was actually exchanged
    assert sum(r[0] for _, _, res in out for r in res) > 0
