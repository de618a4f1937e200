"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 host-side logic: the
static partition computed independently on each rank through the C ABI covers [0, N)
exactly once (Listing 1), and exchanging per-rank spike bitmaps (all-gather)
and decoding them with the library gives every rank the same union (Fig. 2)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2102_04681_b200 import spice as S
        Sw = S.default_slice_width(N, world)
        n_own = S.partition_owned_count(N, rank, world, Sw)
        owned = np.array([S.partition_local_to_global(i, rank, world, Sw) for i in range(n_own)], dtype=np.int64)
        # partition: gather owned sets, check exact cover
        sizes = [None] * world
        dist.all_gather_object(sizes, int(n_own))
        allowned = [None] * world
        dist.all_gather_object(allowned, owned.tolist())
        cover = np.sort(np.concatenate([np.array(x) for x in allowned]))
        ok_cover = np.array_equal(cover, np.arange(N))
        # exchange: random spikes of owned neurons as a bitmap of W words (W from rank 0)
        W = (S.partition_owned_count(N, 0, world, Sw) + 31) // 32
        rng = np.random.default_rng(100 + rank)
        local = np.sort(rng.choice(n_own, size=n_own // 7, replace=False))
        bm = np.zeros(W, dtype=np.uint32)
        for i in local:
            bm[i >> 5] |= np.uint32(1 << (i & 31))
        mine = torch.from_numpy(bm.view(np.int32).copy())
        gathered = [torch.zeros(W, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(gathered, mine)
        words = np.concatenate([g.numpy().view(np.uint32) for g in gathered])
        ids = S.decode_bitmaps(words, world, W, Sw)
        spikes_global = owned[local]
        allsp = [None] * world
        dist.all_gather_object(allsp, spikes_global.tolist())
        union = np.sort(np.concatenate([np.array(x, dtype=np.int64) for x in allsp]))
        ok_union = np.array_equal(ids.astype(np.int64), union)
        # every rank decodes the same list
        lists = [None] * world
        dist.all_gather_object(lists, ids.tolist())
        ok_same = all(l == lists[0] for l in lists)
        # max-over-ranks timing reduction as bench.py does it
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, ok_cover, ok_union, ok_same, t.item(), max(sizes) - min(sizes) <= Sw))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.parametrize("N", [100_003, 4_000])
def test_gloo_two_ranks_partition_and_exchange(N):
    from paper_2102_04681_b200 import build as B
    B.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert len(r) == 6, r
        rank, ok_cover, ok_union, ok_same, tmax, balanced = r
        assert ok_cover and ok_union and ok_same and balanced
        assert tmax == float(world)
