"""Multi-process check of the distributed path (run under torchrun): sharded build + exchange
(dist.build_distributed), each rank's share of the pairs, gather + device sort on rank 0,
compared with the CPU oracle.  Test hook: BENCH_DIST_BACKEND=gloo runs every rank on one GPU.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_check.py [C1 ...]
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1102_1003_b200.dist import build_distributed, gather_triples  # noqa: E402
from paper_1102_1003_b200 import batmap  # noqa: E402
from workloads import make_config  # noqa: E402


def main():
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ.get("BENCH_FORCE_DEVICE", os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group(backend)
    ok = True
    for name in sys.argv[1:] or ["C1", "C3"]:
        w = make_config(name)
        off = torch.as_tensor(w.offsets).cuda()
        tids = torch.as_tensor(w.tids).cuda()
        for max_loop in (0, 1):
            c = build_distributed(off, tids, w.m, seed=5, max_loop=max_loop)
            local = c.pair_supports(threshold=w.threshold, part=rank, n_parts=world)
            allp = gather_triples(local if backend == "nccl" else local.cpu())
            if rank == 0:
                got = batmap.sort_triples(allp.cuda()).cpu().numpy().astype(np.uint32)
                ref = oracle.pairs_merge(w.offsets, w.tids, threshold=w.threshold)
                same = bool(np.array_equal(got, ref))
                ok &= same
                print(f"{name} max_loop={max_loop} world={world} failures={c.info()['n_failures']} "
                      f"K={got.shape[0]} exact={same}", flush=True)
            c.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
