"""Build one config's BatMaps `--n` times (for ncu launch lists / captures of ★K1).

    python tools/build_once.py C4 [--n 2] [--pairs]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_1003_b200 import Collection  # noqa: E402
from workloads import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--n", type=int, default=2)
ap.add_argument("--pairs", action="store_true")
a = ap.parse_args()
w = make_config(a.config)
off = torch.as_tensor(w.offsets).cuda()
tids = torch.as_tensor(w.tids).cuda()
for _ in range(a.n):
    with Collection(off, tids, w.m, seed=1) as c:
        if a.pairs:
            c.pair_supports(threshold=w.threshold)
        st = c.stats()
torch.cuda.synchronize()
print(a.config, {k: round(v, 3) for k, v in st.items() if k.endswith("_ms")})
