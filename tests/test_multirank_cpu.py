"""World-size-2 (and 3) gloo tests of the multi-GPU host logic, on CPU.

Each rank asks the library for its tiles (kde_shard_tiles / kde_shard_tile: round-robin chunks of
tile ids), enumerates the pairs i<j of its tiles through the library's tile map (kde_tile_coords,
Eq. 42-43), and sums an exact
integer weight per pair.  The ranks all-reduce (gloo, int64 SUM) exactly like the GPU path
all-reduces its int64 fixed-point limbs; the result must equal the closed-form total over all
pairs, i.e. the shards cover every pair exactly once."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1505_01998_b200 as kb


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _weight(i, j):
    return (i * 7919 + j * 104729) % 1000003


def _rank_sum(kind, n, d, rank, world):
    T, tot, cnt, chunk = kb.shard_tiles(kind, n, d, rank, world)
    s = 0
    pairs = 0
    ids = [kb.shard_tile(i, rank, world) for i in range(cnt)]
    for t in ids:
        l, q = kb.tile_coords(t)
        rows = np.arange(q * T, min((q + 1) * T, n))
        cols = np.arange(l * T, min((l + 1) * T, n))
        if rows.size == 0 or cols.size == 0:
            continue
        I, J = np.meshgrid(rows, cols, indexing="ij")
        m = J > I
        w = (I[m] * 7919 + J[m] * 104729) % 1000003
        s += int(w.sum())
        pairs += int(m.sum())
    return s, pairs, (ids, tot)


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for kind, n, d in cases:
        s, pairs, rng = _rank_sum(kind, n, d, rank, world)
        t = torch.tensor([s, pairs], dtype=torch.int64)
        dist.all_reduce(t)                              # exact integer combine
        ranges = [None] * world
        dist.all_gather_object(ranges, rng)
        out.append((int(t[0]), int(t[1]), ranges))
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shards_cover_every_pair_once(world):
    cases = [(kb.SUM_PSI6, 1000, 1), (kb.SUM_PSI4, 5000, 1), (kb.SUM_LSCV_h, 1300, 2), (kb.SUM_LSCV_H, 1100, 4)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = q.get(timeout=600)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (kind, n, d), (s, pairs, ranges) in zip(cases, res):
        i, j = np.triu_indices(n, 1)
        assert pairs == n * (n - 1) // 2
        assert s == int(((i * 7919 + j * 104729) % 1000003).sum())
        # disjoint and covering every tile id exactly once
        allids = sorted(t for ids, _ in ranges for t in ids)
        assert allids == list(range(ranges[0][1]))
