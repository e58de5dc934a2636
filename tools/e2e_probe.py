"""Diagnostics: the bench's sequence (device-timed builds, then batmap_mine_host calls) with
BATMAP_TRACE=2 timestamps inside the K2 plan upload; prints each mine_host call's wall time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1102_1003_b200 import Collection, mine_host  # noqa: E402
from workloads import make_config  # noqa: E402

w = make_config("C4")
off_d, tids_d = torch.as_tensor(w.offsets).cuda(), torch.as_tensor(w.tids).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    with Collection(off_d, tids_d, w.m, seed=1) as c:
        c.pair_supports(threshold=w.threshold)
    print("device build+pairs", i, flush=True)
off_h = torch.from_numpy(np.ascontiguousarray(w.offsets)).pin_memory()
tids_h = torch.from_numpy(np.ascontiguousarray(w.tids)).pin_memory()
for i in range(7):
    flush.zero_()
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = mine_host(off_h.numpy(), tids_h.numpy(), w.m, threshold=w.threshold, seed=1, capacity=30000)
    torch.cuda.synchronize()
    print("mine_host %d wall ms %.1f" % (i, (time.perf_counter() - t) * 1e3), flush=True)
