"""The NCCL branches of the multi-GPU path, on the one GPU this build has: a world-size-1 NCCL
process group.  Every multi-rank test shares one GPU over gloo (NCCL refuses two ranks on one
device), which stages through host memory; this runs the branches the 8-GPU box takes instead --
all_gather_into_tensor of the BatMap words and failure records (dist._all_gather_flat), the
device-resident all_gather / gather of the triples (dist.gather_triples), the device merge-sort,
bench.py's pre-timing verification -- and checks the triples against the CPU oracle.  (A one-part
build is the whole build, so build_distributed exchanges nothing at world 1; _all_gather_flat is
called directly.)  It proves
the tensor shapes, dtypes and devices the NCCL calls get, not the multi-rank exchange itself
(that is covered, with host staging, by test_gpu_dist.py and test_dist_gloo.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        import bench
        import oracle
        from paper_1102_1003_b200.dist import (_all_gather_flat, build_distributed, mine_distributed,
                                               pair_supports_distributed)
        from workloads import zipf

        assert dist.get_backend() == "nccl"
        out = {}
        m = 6000
        off, tids = zipf(700, m, seed=11)
        ref = oracle.pairs_merge(off, tids, threshold=2).astype(np.int64)
        got = mine_distributed(torch.as_tensor(off).pin_memory(), torch.as_tensor(tids).pin_memory(), m,
                               threshold=2, seed=3, max_loop=1)
        out["mine"] = bool(np.array_equal(np.asarray(got, np.int64), ref))
        coll = build_distributed(torch.as_tensor(off).to(dev), torch.as_tensor(tids).to(dev), m, seed=5,
                                 max_loop=2)
        res = pair_supports_distributed(coll, threshold=2)
        coll.close()
        out["pairs"] = bool(np.array_equal(res.cpu().numpy().astype(np.int64), ref))
        out["bench_verify"] = bool(bench._verify_small_instance(dev, "nccl", 0, 1))
        # the exchange of the sharded build (a world-1 build has none): the BatMap words (int32)
        # and failure records (int64) through all_gather_into_tensor, device to device
        ok = True
        for dt in (torch.int32, torch.int64):
            x = torch.arange(1000, dtype=dt, device=dev) * 7 - 3
            y = _all_gather_flat(x)
            ok = ok and y.is_cuda and y.dtype == dt and torch.equal(y, x)
        out["all_gather_flat"] = bool(ok)
        out["n_ref"] = int(ref.shape[0])
        q.put(("ok", out))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_world1_branches_equal_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_free_port(), q))
    p.start()
    status, out = q.get(timeout=600)
    p.join(timeout=60)
    assert status == "ok", out
    assert out["n_ref"] > 0 and out["mine"] and out["pairs"] and out["bench_verify"] and out["all_gather_flat"], out
