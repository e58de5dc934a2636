"""Multi-rank host logic on CPU (gloo, world_size 2): the tile partition, the flat all_gather of
the sharded build's exchange and the gather of compacted triples that the N-GPU path uses
(SURVEY §8(e)).  The GPU parts (per-rank pair
supports, device merge-sort) are covered by tests/test_gpu_parity.py::test_items_subset_and_parts."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1102_1003_b200 import plan_work
        from paper_1102_1003_b200.dist import gather_triples
        import oracle
        from workloads import uniform

        # 1) the planner's share of this rank: gather every rank's tiles and check exact cover
        class_n, class_w = [7800, 2200], [1536, 3072]
        items, wc, work = plan_work(class_n, class_w, rank, world)
        # (tile key, tile column, k-chunks) per work item; tiles may be cut into k pieces
        t = torch.as_tensor(np.stack([items[:, 0] * 100000 + items[:, 1] * 1000 + items[:, 2], items[:, 3],
                                      items[:, 5] - items[:, 4]], 1).astype(np.int32))
        allt = gather_triples(t)
        w = torch.tensor([work], dtype=torch.int64)
        ws = [torch.zeros_like(w) for _ in range(world)]
        dist.all_gather(ws, w)
        # 2) triples: each rank owns a disjoint share of the oracle's pairs (rows dealt round-robin)
        off, tids = uniform(120, 4000, 0.05, 3)
        full = oracle.pairs_merge(off, tids, threshold=3).astype(np.int32)
        mine = full[full[:, 0] % world == rank]
        got = gather_triples(torch.as_tensor(mine))
        empty = gather_triples(torch.zeros((0, 3), dtype=torch.int32))  # empty parts are legal
        # 3) the flat all_gather of the sharded build's exchange (dist.build_distributed)
        from paper_1102_1003_b200.dist import _all_gather_flat

        flat = _all_gather_flat(torch.arange(5, dtype=torch.int64) + 10 * rank)
        flat_ok = flat.tolist() == [10 * r + k for r in range(world) for k in range(5)]
        if not flat_ok:
            raise AssertionError(f"all_gather_flat: {flat.tolist()}")
        if rank == 0:
            g = got.numpy()
            g = g[np.lexsort((g[:, 1], g[:, 0]))]
            a = allt.numpy()
            cover = (len({(int(x), int(y)) for x, y, _ in a}), int(a[:, 2].sum()))
            q.put(("ok", cover, [int(x) for x in ws], bool(np.array_equal(g, full)), empty.shape[0]))
        else:
            q.put(("ok", None if got is None else -1, None, got is None, None if empty is None else -1))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


def test_gather_and_partition_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[0] == "ok" for r in res), res
    r0 = [r for r in res if r[1] is not None and r[1] != -1][0]
    from paper_1102_1003_b200 import plan_work

    full = plan_work([7800, 2200], [1536, 3072], 0, 1)[0]
    n_tiles = len({(int(a) * 100000 + int(b) * 1000 + int(ti), int(tj)) for a, b, ti, tj in full[:, :4]})
    assert r0[1] == (n_tiles, int((full[:, 5] - full[:, 4]).sum()))  # the ranks cover every tile and chunk once
    assert abs(r0[2][0] - r0[2][1]) <= 128 * 128 * 3072  # balanced within one tile
    assert r0[3] is True  # gathered triples == the full result
    assert r0[4] == 0
    others = [r for r in res if r is not r0]
    assert all(r[3] is True for r in others)  # non-destination ranks get None
