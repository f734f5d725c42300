"""Multi-process (world 2 and 4, gloo on CPU) test of the sharding logic.

The library's host planner (qsim_plan_make_local / qsim_plan_canonical_globals,
dist.cu) decides which shard exchanges bring global qubits local and how the
logical -> physical map changes.  Here each rank holds its shard as a numpy
array, the planned steps are executed with the exchange the library performs
(rank r swaps the half of its shard whose top local bit differs from its bit g
with rank r ^ 2^(g - nl); or the all-to-all that swaps
every global position with the top local positions at once), and the
re-assembled state must equal the original state read through the map.  No GPU is involved.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _logical_state(shards, pos, n, nl):
    """Re-assemble the logical state from shards + map."""
    out = np.empty(1 << n, complex)
    for r, sh in enumerate(shards):
        for i in range(sh.size):
            P = (r << nl) | i
            x = 0
            for q in range(n):
                x |= ((P >> pos[q]) & 1) << (n - 1 - q)
            out[x] = sh[i]
    return out


def _swap_local_bits(sh, p1, p2):
    idx = np.arange(sh.size)
    b1, b2 = (idx >> p1) & 1, (idx >> p2) & 1
    j = idx & ~((1 << p1) | (1 << p2)) | (b2 << p1) | (b1 << p2)
    out = np.empty_like(sh)
    out[j] = sh
    return out


def _worker(rank, world, port, n, seqs, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from paper_quant_ph_0201042_b200 import qsim as Q
    try:
        kg = world.bit_length() - 1
        nl = n - kg
        rng = np.random.default_rng(7)
        full = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        shard = full[rank << nl:(rank + 1) << nl].copy()
        pos = np.array([n - 1 - q for q in range(n)], np.int32)

        def run(steps, shard):
            for kind, a, b in steps:
                if kind == 0:
                    shard = _swap_local_bits(shard, a, b)
                elif kind == 2:
                    # all-to-all: block j (top a local bits) -> rank j, block rank <- rank j's block
                    blk = shard.size >> a
                    out = shard.copy()
                    reqs, bufs = [], {}
                    for p in range(world):
                        if p == rank:
                            continue
                        send = torch.from_numpy(np.ascontiguousarray(shard[p * blk:(p + 1) * blk]).view(np.float64).copy())
                        bufs[p] = torch.empty_like(send)
                        reqs += [dist.isend(send, p), dist.irecv(bufs[p], p)]
                    for r_ in reqs:
                        r_.wait()
                    for p, t in bufs.items():
                        out[p * blk:(p + 1) * blk] = t.numpy().view(complex)
                    shard = out
                else:
                    gb = a - nl
                    partner = rank ^ (1 << gb)
                    bit = (rank >> gb) & 1
                    half = shard.size // 2
                    mine = shard[(1 - bit) * half:(2 - bit) * half]
                    send = torch.from_numpy(np.ascontiguousarray(mine).view(np.float64).copy())
                    recv = torch.empty_like(send)
                    reqs = [dist.isend(send, partner), dist.irecv(recv, partner)]
                    for r_ in reqs:
                        r_.wait()
                    shard = shard.copy()
                    shard[(1 - bit) * half:(2 - bit) * half] = recv.numpy().view(complex)
            return shard

        for need in seqs:
            pos2, steps = Q.qsim_plan_make_local(n, world, pos, need)
            assert all(pos2[qq] < nl for qq in need)
            shard = run(steps, shard)
            pos = pos2
        pos3, steps = Q.qsim_plan_canonical_globals(n, world, pos)
        shard = run(steps, shard)
        pos = pos3
        assert all(pos[qq] == n - 1 - qq for qq in range(n) if pos[qq] >= nl)
        # gather and check
        t = torch.from_numpy(shard.view(np.float64).copy())
        allt = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        shards = [x.numpy().view(complex) for x in allt]
        got = _logical_state(shards, pos, n, nl)
        ok = np.array_equal(got, full)
        q.put((rank, bool(ok), ""))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,seqs", [
    (2, 6, [[0], [1, 0], [5], [0, 3]]),
    (4, 7, [[0, 1], [1], [2, 0, 6], [3, 4, 5]]),
    (4, 5, [[0, 1, 2], [3, 4], [1]]),
    (8, 7, [[0, 1, 2], [3], [0, 4, 5], [6, 1]]),
    (4, 6, [[0, 1], [2, 3], [0, 5]]),
])
def test_sharded_exchanges_preserve_the_state(world, n, seqs):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, seqs, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
