"""Query sharding across GPUs.

Every rank holds the full reference tree (rebuilt locally; the device build is
deterministic, so trees are bit-identical across ranks) and processes the
query blocks ``rank, rank + world, rank + 2*world, ...`` -- a round-robin deal
of the (<= 64-point) blocks in tree order, i.e. a spatially uniform sample per
rank, which balances the strongly density-dependent per-block cost.  Each
rank writes only its blocks' queries into a zero vector; one collective sum
over these disjoint supports assembles the full result exactly (x + 0 == x),
which is the gather of the north star.
"""

from __future__ import annotations

import numpy as np


def shard_blocks(nblocks: int, rank: int, world: int):
    """(begin, end, stride) of the query blocks owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return rank, nblocks, world


def query_block_ranges(start, end, left, right, limit: int = 64):
    """Host restatement of the engine's query blocks (fg_traverse.cu:
    block_ranges, mode 0): the maximal tree nodes with <= ``limit`` points, in
    tree order; leaves larger than ``limit`` are cut into runs of ``limit``.
    Takes the preorder node arrays of ``KdTree.arrays()``."""
    out = []
    stack = [0]
    while stack:
        v = stack.pop()
        cnt = int(end[v] - start[v])
        if cnt <= limit or left[v] < 0:
            for s in range(0, cnt, limit):
                out.append((int(start[v]) + s, min(limit, cnt - s)))
        else:
            stack.append(int(right[v]))
            stack.append(int(left[v]))
    return out


def owned_queries(ranges, perm, rank: int, world: int):
    """Original query indices processed by ``rank`` under ``shard_blocks``."""
    b0, b1, stride = shard_blocks(len(ranges), rank, world)
    idx = [np.arange(s, s + c) for s, c in ranges[b0:b1:stride]]
    pos = np.concatenate(idx) if idx else np.zeros(0, np.int64)
    return np.asarray(perm)[pos]


def gather_disjoint(values, group=None):
    """Assemble per-rank vectors with disjoint supports (collective sum)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(values, op=dist.ReduceOp.SUM, group=group)
    return values


def run_sharded(config, qtree, rtree, out, rank: int, world: int, group=None):
    """Run ``config.algorithm`` on this rank's query blocks, then gather.

    ``out`` is a float64 tensor of length M on this rank's device (zeroed
    here).  Returns the local ResultVector (counters of this rank's shard).
    """
    from .summation_engine import query_block_count, run_blocks

    nb = query_block_count(qtree)
    b0, b1, stride = shard_blocks(nb, rank, world)
    out.zero_()
    res = run_blocks(config, qtree, rtree, b0, b1, stride, out=out)
    gather_disjoint(out, group)
    return res


def run_sharded_sweep(config, qtree, rtree, bandwidths, out, rank: int, world: int, group=None):
    """The whole bandwidth sweep on this rank's query blocks (one engine call,
    one traversal launch), then ONE collective over all bandwidths' values.

    ``out`` is a float64 tensor (len(bandwidths), M) on this rank's device
    (zeroed here).  Returns this rank's ResultVectors.
    """
    from .summation_engine import query_block_count, sweep_run

    nb = query_block_count(qtree)
    out.zero_()
    res = sweep_run(config, qtree, rtree, bandwidths, out=out,
                    block_range=shard_blocks(nb, rank, world))
    gather_disjoint(out, group)
    return res
