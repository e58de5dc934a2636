"""Time the BatMap build (★K1) alone on BASELINE configs: best of `reps` builds, phase split from
the library's CUDA events.  One JSON line per config.

    python tools/build_bench.py [--reps 5] C2 C5_p0.1 ...
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1102_1003_b200 import Collection  # noqa: E402
from workloads import make_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("configs", nargs="*", default=["C2", "C3", "C4", "C5_p0.01", "C5_p0.1"])
    a = ap.parse_args()
    for name in a.configs:
        w = make_config(name)
        off_d = torch.as_tensor(w.offsets).cuda()
        tids_d = torch.as_tensor(w.tids).cuda()
        best = None
        for _ in range(a.reps):
            torch.cuda.synchronize()
            c = Collection(off_d, tids_d, w.m, seed=1)
            st, inf = c.stats(), c.info()
            c.close()
            if best is None or st["build_ms"] < best[0]["build_ms"]:
                best = (st, inf)
        st, inf = best
        print(json.dumps(dict(config=name, tier=os.environ.get("BATMAP_K1_SMALL", "cluster"), nnz=w.nnz,
                              build_ms=st["build_ms"], k1_insert_ms=st["k1_insert_ms"],
                              k1_encode_ms=st["k1_encode_ms"], failures=inf["n_failures"],
                              arena_MB=inf["arena_bytes"] / 1e6,
                              insertions_per_s=2 * w.nnz / (st["k1_insert_ms"] / 1e3))), flush=True)


if __name__ == "__main__":
    main()
