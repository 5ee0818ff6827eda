"""World-size-2 multi-process test of the sharding host logic over gloo on CPU
(DESIGN.md §5): flop-balanced split, per-rank shard build + partial cutsize
(CPU oracle standing in for the per-rank GPU build), allreduce of the
partials, concatenation of shards == single-rank graph."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1710_07769_b200.dist import allreduce_cut, shard_bounds, split_points
from rig_inputs import make_small


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = make_small(cfg)
        cp = oracle.transpose(w.n, w.n, w.row_ptr, w.col_idx, w.val)[0]
        f, P = oracle.row_products(w.row_ptr, w.col_idx, cp)
        pre = np.concatenate([[0], np.cumsum(f)])
        split = split_points(pre, world)
        rb, re = shard_bounds(split, rank)
        g = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=w.scale_rows, drop_tol=w.drop_tol,
                         row_begin=rb, row_end=re)
        part_cut = oracle.cutsize(g.row_ptr, g.col, g.w, w.part, w.K, row_begin=rb)[0]
        cut = torch.tensor([part_cut], dtype=torch.float64)
        allreduce_cut(cut)
        shards = [None] * world
        dist.all_gather_object(shards, (rb, re, g.col.tolist(), g.w.tolist(), g.products))
        q.put((rank, split, float(cut[0]), shards))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [2, 5])
def test_sharded_build_and_allreduce_world2(cfg):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    res.sort()
    w = make_small(cfg)
    full = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=w.scale_rows, drop_tol=w.drop_tol)
    full_cut = oracle.cutsize(full.row_ptr, full.col, full.w, w.part, w.K)[0]
    splits = {tuple(r[1]) for r in res}
    assert len(splits) == 1  # every rank derives the same split, no communication
    split = list(splits.pop())
    assert split[0] == 0 and split[-1] == w.n
    # flop balance: each shard within one row's products of P / world
    shards = res[0][3]
    prods = [s[4] for s in shards]
    assert abs(prods[0] - prods[1]) <= 2 * max(np.diff(w.row_ptr)) * 64 + 0.01 * sum(prods)
    for r in res:  # the allreduced cut is identical on every rank and equals the full one
        assert abs(r[2] - full_cut) <= 1e-12 * full_cut
    cols = np.concatenate([np.array(s[2], dtype=np.int32) for s in shards])
    ws = np.concatenate([np.array(s[3], dtype=np.float64) for s in shards])
    np.testing.assert_array_equal(cols, full.col)
    assert ws.tobytes() == full.w.tobytes()


def test_split_points_matches_definition():
    rng = np.random.default_rng(3)
    f = rng.integers(0, 50, 1000)
    pre = np.concatenate([[0], np.cumsum(f)])
    for parts in (1, 2, 3, 8):
        sp = split_points(pre, parts)
        P = pre[-1]
        for g in range(parts):
            assert sp[g] == int(np.searchsorted(pre, -(-g * P // parts), side="left"))
        assert sp[-1] == 1000 and sp == sorted(sp)
