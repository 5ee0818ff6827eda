"""The multi-GPU product path (local
subgraphs per processor) executed for real: two processes, one shard each,
every shard built by librig through dist.build_cut_sharded (flop-balanced
split on the device, rig_build_cut per shard, all_reduce of the partial cuts).
Only one GPU exists on the test box, so both ranks share cuda:0 and talk over
gloo (which reduces CUDA tensors through the host); the ranks' kernels never
wait on each other, only the 8-byte allreduce joins them.  The concatenated
shards must equal the oracle's single-rank graph bit for bit and the reduced
cut must match the oracle's within 1e-12."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import oracle  # noqa: E402
from rig_inputs import make_small  # noqa: E402

REL = 1e-12


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1710_07769_b200 import dist as rdist
        from paper_1710_07769_b200 import rig

        w = make_small(cfg)
        A = rig.CSR(w.row_ptr, w.col_idx, w.val)
        part = torch.as_tensor(w.part, device="cuda")
        g, cut, (rb, re) = rdist.build_cut_sharded(A, part, w.K, w.scale_rows, w.drop_tol)
        torch.cuda.synchronize()
        shard = (rb, re, g.row_ptr.cpu().numpy(), g.col_idx.cpu().numpy(), g.w.cpu().numpy())
        shards = [None] * world
        dist.all_gather_object(shards, shard)
        q.put((rank, float(cut.item()), shards))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [2, 4, 5])
def test_sharded_product_path_world2(cfg):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for rank, cut, shards in res:
        assert shards is not None, cut
    w = make_small(cfg)
    orc = oracle.build(w.row_ptr, w.col_idx, w.val, scale_rows=w.scale_rows, drop_tol=w.drop_tol)
    ocut = oracle.cutsize(orc.row_ptr, orc.col, orc.w, w.part, w.K)[0]
    shards = res[0][2]
    assert shards[0][0] == 0 and shards[-1][1] == w.n and shards[0][1] == shards[1][0]
    assert 0 < shards[0][1] < w.n  # both ranks got rows
    rp = [shards[0][2]] + [s[2][1:] + shards[0][2][-1] for s in shards[1:]]
    np.testing.assert_array_equal(np.concatenate(rp), orc.row_ptr)
    np.testing.assert_array_equal(np.concatenate([s[3] for s in shards]), orc.col)
    assert np.concatenate([s[4] for s in shards]).tobytes() == orc.w.tobytes()
    for rank, cut, _ in res:  # the allreduced cut, on every rank
        assert abs(cut - ocut) <= REL * abs(ocut)
    assert res[0][1] == res[1][1]
