"""Query sharding across GPUs.

Every rank holds the full reference tree (rebuilt locally; the device build is
deterministic, so trees are bit-identical across ranks) and processes the
query blocks ``rank, rank + world, rank + 2*world, ...`` -- a round-robin deal
of the (<= 64-point) blocks in tree order, i.e. a spatially uniform sample per
rank, which balances the strongly density-dependent per-block cost.  Blocks
are even runs of <= 64 tree-order points inside the maximal nodes of <=
max(64, min(4096, n / 16)) points (``query_block_ranges`` restates the rule).  Each
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


QBLOCK = 64          # points per query block (fg_traverse_kernel.cuh: kQBlock)
QBLOCK_NODE = 4096   # node-size cap of the block cut (fg_traverse.cu: kQBlockNode)


def query_block_ranges(start, end, left, right, limit: int = QBLOCK):
    """Host restatement of the engine's query blocks (fg_traverse.cu:
    block_marks_kernel + the scan that numbers the runs): every maximal tree
    node with <= lim = max(64, min(4096, n // 16)) points (or a leaf of any
    size) is cut into ceil(count / 64) runs of consecutive tree-order points,
    as even as possible (run r covers [count*r // k, count*(r+1) // k)).
    Returns (start, count) per block in tree order.  Takes the preorder node
    arrays of ``KdTree.arrays()`` (or the oracle's export); node 0 is the
    root.  ``fg_query_block_ranges`` returns the same list (gpu test)."""
    start = np.asarray(start)
    end = np.asarray(end)
    left = np.asarray(left)
    right = np.asarray(right)
    n = int(end[0] - start[0])
    lim = max(limit, min(QBLOCK_NODE, n // 16))
    out = []

    def emit(v):
        cnt = int(end[v] - start[v])
        k = (cnt + limit - 1) // limit
        for r in range(k):
            s0, s1 = cnt * r // k, cnt * (r + 1) // k
            out.append((int(start[v]) + s0, s1 - s0))

    stack = [0]
    while stack:
        v = stack.pop()
        if int(end[v] - start[v]) <= lim or left[v] < 0:
            emit(v)
        else:
            stack.append(int(right[v]))
            stack.append(int(left[v]))
    out.sort()
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
    here on torch's current stream, which the engine call then runs on).
    Returns the local ResultVector (counters of this rank's shard).
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
    (zeroed here on torch's current stream, which the engine call then runs
    on).  Returns this rank's ResultVectors.
    """
    from .summation_engine import query_block_count, sweep_run

    nb = query_block_count(qtree)
    out.zero_()
    res = sweep_run(config, qtree, rtree, bandwidths, out=out,
                    block_range=shard_blocks(nb, rank, world))
    gather_disjoint(out, group)
    return res
