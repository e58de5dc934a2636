import sys, time, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1102_1003_b200 import mine_host
from workloads import make_config
w = make_config("C4")
off_h = torch.from_numpy(np.ascontiguousarray(w.offsets)).pin_memory(); tids_h = torch.from_numpy(np.ascontiguousarray(w.tids)).pin_memory()
off_np, tids_np = off_h.numpy(), tids_h.numpy()
for i in range(4):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = mine_host(off_np, tids_np, w.m, threshold=w.threshold, seed=1, capacity=30000)
    torch.cuda.synchronize(); print("mine_host wall ms %.1f" % ((time.perf_counter() - t) * 1e3), r.shape, flush=True)
