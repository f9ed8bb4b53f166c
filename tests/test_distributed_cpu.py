"""Multi-rank query sharding on CPU (gloo, world_size 2).

The engine itself needs a GPU; these tests exercise the host-side sharding
logic of paper_1206_6857_b200.distributed -- the engine's own query-block
partition (``query_block_ranges`` restates fg_traverse.cu's block rule; a gpu
test pins it to ``fg_query_block_ranges``) dealt round-robin to ranks -- with
the CPU oracle's DFS DITO standing in for each rank's per-shard compute: the
deal covers every query exactly once, the collective sum over disjoint
supports assembles the full vector exactly, and every query is within eps.
"""

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
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_path):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_1206_6857_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(5)
    pts = rng.random((3000, 3))
    w = rng.uniform(0.5, 1.5, 3000)
    tree = oracle.Tree(pts, w, 25)
    ex = tree.export()
    ranges = D.query_block_ranges(ex["start"], ex["end"], ex["left"], ex["right"])
    mine = D.owned_queries(ranges, ex["perm"], rank, world)
    vals = torch.zeros(pts.shape[0], dtype=torch.float64)
    hits = torch.zeros(pts.shape[0], dtype=torch.float64)
    if mine.size:
        tree.refresh_moments(0.1, 6)
        v, _ = oracle.run_sharded("dito", pts[mine], tree, 0.1, 0.01, threads=1)
        vals[torch.from_numpy(mine)] = torch.from_numpy(v)
        hits[torch.from_numpy(mine)] = 1.0
    D.gather_disjoint(vals)
    D.gather_disjoint(hits)
    if rank == 0:
        full = oracle.naive_sum(pts, pts, w, 0.1)
        np.save(result_path, np.stack([vals.numpy(), full, hits.numpy()]))
    dist.barrier()
    dist.destroy_process_group()


def test_blocks_partition_queries():
    import oracle
    from paper_1206_6857_b200 import distributed as D

    rng = np.random.default_rng(1)
    for n, leaf in ((1, 25), (31, 25), (1000, 25), (5000, 10), (700, 1)):
        pts = rng.random((n, 2))
        t = oracle.Tree(pts, None, leaf)
        ex = t.export()
        ranges = D.query_block_ranges(ex["start"], ex["end"], ex["left"], ex["right"])
        assert all(1 <= c <= 64 for _, c in ranges)
        # every block lies inside one maximal node of <= lim points (or a leaf)
        lim = max(64, min(4096, n // 16))
        size = ex["end"] - ex["start"]
        for s, c in ranges:
            inside = (ex["start"] <= s) & (s + c <= ex["end"])
            assert np.any(inside & ((size <= lim) | (ex["left"] < 0)))
        pos = np.concatenate([np.arange(s, s + c) for s, c in ranges])
        np.testing.assert_array_equal(pos, np.arange(n))  # tree order, exact cover
        for world in (1, 2, 3, 8):
            owned = np.concatenate([D.owned_queries(ranges, ex["perm"], r, world)
                                    for r in range(world)])
            assert sorted(owned.tolist()) == list(range(n))


def test_shard_blocks_validation():
    from paper_1206_6857_b200 import distributed as D

    assert D.shard_blocks(10, 1, 4) == (1, 10, 4)
    with pytest.raises(ValueError):
        D.shard_blocks(10, 4, 4)


def test_gloo_world2_gather_matches_full(tmp_path):
    out = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got, full, hits = np.load(out)
    np.testing.assert_array_equal(hits, np.ones_like(hits))  # every query exactly once
    assert np.max(np.abs(got - full) / full) <= 0.01
