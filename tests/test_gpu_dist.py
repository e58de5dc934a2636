"""The multi-GPU public path end to end, two ranks sharing one GPU over gloo (the test hook the
bench uses on a one-GPU box): dist.mine_distributed = H2D of the CSR on every rank, sharded
build + exchange (batmap_build_shard / shard_export / shard_import), this rank's share of the
pairs (batmap_pair_supports_part), gather and device sort on rank 0, D2H.  Rank 0's triples
must equal the oracle's; the other rank gets None."""
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


def _worker(rank, world, port, max_loop, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1102_1003_b200.dist import mine_distributed
        from workloads import zipf

        torch.cuda.set_device(0)
        off, tids = zipf(700, 6000, seed=11)
        m = 6000
        got = mine_distributed(torch.as_tensor(off).pin_memory(), torch.as_tensor(tids).pin_memory(), m,
                               threshold=2, seed=3, max_loop=max_loop)
        if rank == 0:
            ref = oracle.pairs_merge(off, tids, threshold=2).astype(np.int64)
            q.put(("ok", bool(np.array_equal(np.asarray(got, np.int64), ref)), int(ref.shape[0])))
        else:
            q.put(("ok", got is None, 0))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,max_loop", [(2, 0), (3, 1)])
def test_mine_distributed_equals_oracle(world, max_loop):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, max_loop, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[0] == "ok" and r[1] is True for r in res), res
    assert max(r[2] for r in res) > 0
