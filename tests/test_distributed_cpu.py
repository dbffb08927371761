"""CPU (gloo, world_size 2): the multi-GPU host logic — fused statistics
all-reduce (bit-exact integer sums through the int64 view), per-rank send
counts derived from the permutation's key_offsets, count exchange — on the
same code paths bench.py / a2a.py use with NCCL on the B200s."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp_

from paper_2604_23150_b200.distributed import (all_reduce_stats, exchange_counts,
                                               gather_shards, groups_per_rank, rank_of_group,
                                               send_counts_from_offsets, shard_bounds)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        big = (1 << 62) + rank  # beyond int32; exercises the u64->i64 view
        stats = torch.tensor([big, 7 * (rank + 1), 0], dtype=torch.uint64)
        all_reduce_stats(stats)
        sc = torch.tensor([rank * 10 + r for r in range(world)], dtype=torch.int64)
        rc = exchange_counts(sc)
        # sharded scoring: each rank fills its candidate rows, then all-gather
        P, L = 6, 3
        lo, hi = shard_bounds(P, world, rank)
        fin = torch.full((P * L, 4), -1.0, dtype=torch.float64)
        for p in range(lo, hi):
            fin[p * L:(p + 1) * L] = torch.arange(4, dtype=torch.float64) / 3 + p
        gather_shards(fin, (hi - lo) * L)
        q.put((rank, [int(x) for x in stats.tolist()], rc.tolist(), fin.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_gloo_stats_allreduce_and_count_exchange():
    world = 2
    port = _free_port()
    ctx = mp_.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict((r, (s, c, f)) for r, s, c, f in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = [((1 << 62) * 2 + 1) % (1 << 64), 7 + 14, 0]
    full = np.concatenate([np.tile(np.arange(4) / 3 + p, (3, 1)) for p in range(6)])
    for r in range(world):
        assert got[r][0] == expect
        np.testing.assert_array_equal(got[r][2], full)  # every rank holds all candidates
        assert got[r][1] == [src * 10 + r for src in range(world)]


def test_send_counts_from_key_offsets(oracle):
    rng = np.random.default_rng(4)
    T, E, D, k = 3000, 64, 8, 4
    idx = np.argsort(rng.random((T, E)), axis=1)[:, :k].astype(np.int32)
    src = rng.integers(0, D, T).astype(np.uint32)
    groups = [list(range(d * 8, d * 8 + 8)) for d in range(D)]
    g2n = [d // 4 for d in range(D)]
    lut = oracle.dest_lut(groups, g2n, E)
    lay = oracle.dispatch_layout(idx, src, lut, D, E, g2n)
    dest = lut[np.array(g2n)[src][np.arange(T * k) // k], idx.reshape(-1)]
    for world in (1, 2, 4, 8):
        counts = send_counts_from_offsets(lay["key_offsets"], D, E, world)
        ranks = np.array([rank_of_group(int(g), D, world) for g in dest])
        np.testing.assert_array_equal(counts, np.bincount(ranks, minlength=world))
        assert groups_per_rank(D, world) * world == D
    with pytest.raises(ValueError):
        groups_per_rank(8, 3)
