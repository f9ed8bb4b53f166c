"""Multi-rank query sharding on CPU (gloo, world_size 2).

The engine itself needs a GPU; these tests exercise the host-side sharding
logic of paper_1206_6857_b200.distributed with the CPU oracle standing in for
the per-shard compute: the round-robin block deal covers every query exactly
once, and the collective sum over disjoint supports reproduces the full
result bit-for-bit.
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
    if mine.size:
        vals[torch.from_numpy(mine)] = torch.from_numpy(
            oracle.naive_sum(pts[mine], pts, w, 0.1))
    D.gather_disjoint(vals)
    if rank == 0:
        full = oracle.naive_sum(pts, pts, w, 0.1)
        np.save(result_path, np.stack([vals.numpy(), full]))
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
    got, full = np.load(out)
    np.testing.assert_array_equal(got, full)
