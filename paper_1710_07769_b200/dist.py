"""Multi-GPU plumbing: rows of C sharded over ranks (one process per GPU).

DESIGN.md §5.  Every rank holds the full A (replicated) and the partition;
rows of C are split into contiguous, flop-balanced ranges (rig_row_split, on
the device, identical on every rank, no communication); each rank builds its
shard and its partial cutsize with rig_build_cut; one all_reduce(SUM) of the
8-byte partial over NCCL (torch.distributed) yields the cutsize everywhere.
This is the only collective: the graph shards stay where they were built
(§4: parallel SpGEMM producing local subgraphs).
"""
from __future__ import annotations

import bisect

import torch
import torch.distributed as dist


def split_points(fprefix, parts):
    """Host mirror of the device split rule (k_split): split[g] is the first
    row r with fprefix[r] >= ceil(g * P / parts), split[parts] = n, where
    fprefix is the exclusive prefix of per-row products (length n + 1)."""
    n = len(fprefix) - 1
    P = int(fprefix[-1])
    out = []
    for g in range(parts):
        target = -(-g * P // parts)
        out.append(bisect.bisect_left(list(fprefix), target) if n >= 0 else 0)
    out.append(n)
    return out


def shard_bounds(split, rank):
    return int(split[rank]), int(split[rank + 1])


def allreduce_cut(cut: torch.Tensor, group=None) -> torch.Tensor:
    """a8: sum of the per-rank partial cutsizes (fp64[1]) in place."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(cut, op=dist.ReduceOp.SUM, group=group)
    return cut


def build_cut_sharded(A, part, K, scale_rows=1, drop_tol=0.0, group=None, split=None, flags=0):
    """Each rank: its G_RIP shard + the global cutsize.  Returns
    (graph_shard, cut_tensor, (row_begin, row_end))."""
    from . import rig

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if split is None:
        split = rig.rig_row_split(A, world) if world > 1 else [0, A.nrows]
    rb, re = shard_bounds(split, rank)
    g, cut = rig.rig_build_cut(A, part, K, rb, re, scale_rows, drop_tol, flags)
    allreduce_cut(cut, group)
    return g, cut, (rb, re)
