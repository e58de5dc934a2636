"""Time the BatMap build (★K1) alone on BASELINE configs: best of `reps` builds, phase split from
the library's CUDA events, per K1 variant (environment switches of build.cu, read per build).
With --check, one build per variant is also run through the pair kernels and compared with the
C5 goldens (tests/golden/c5) or the horizontal CPU oracle.  One JSON line per (config, variant).

    python tools/build_bench.py [--reps 5] [--check] [--variants "byte=1;byte=0,small=cluster"] C2 C5_p0.1 ...

Variant keys: byte -> BATMAP_K1_BYTE, small -> BATMAP_K1_SMALL, spread -> BATMAP_K1_SPREAD,
side -> BATMAP_K1_SIDE.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

from paper_1102_1003_b200 import Collection  # noqa: E402
from workloads import make_config  # noqa: E402

ENV = {"byte": "BATMAP_K1_BYTE", "small": "BATMAP_K1_SMALL", "spread": "BATMAP_K1_SPREAD", "side": "BATMAP_K1_SIDE",
       "ipc": "BATMAP_K1_IPC", "stage": "BATMAP_K1_STAGE"}


def _reference(w):
    gold = os.path.join(ROOT, "tests", "golden", "c5", "manifest.json")
    if w.name.startswith("C5_") and os.path.exists(gold):
        from make_goldens import load_triples

        ent = json.load(open(gold))[w.name]
        t = load_triples(os.path.join(ROOT, "tests", "golden", "c5", ent["file"]))
        return t[t[:, 2] >= w.threshold], "golden"
    import oracle

    return oracle.pairs_horizontal(w.offsets, w.tids, w.m, threshold=w.threshold), "horizontal oracle"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--variants", default="byte=1", help="';'-separated variants of ','-separated key=value")
    ap.add_argument("configs", nargs="*", default=["C2", "C3", "C4", "C5_p0.01", "C5_p0.1"])
    a = ap.parse_args()
    for name in a.configs:
        w = make_config(name)
        off_d = torch.as_tensor(w.offsets).cuda()
        tids_d = torch.as_tensor(w.tids).cuda()
        ref = None
        for var in a.variants.split(";"):
            for k in ENV.values():
                os.environ.pop(k, None)
            for kv in var.split(","):
                if kv:
                    k, v = kv.split("=")
                    os.environ[ENV[k]] = v
            Collection(off_d, tids_d, w.m, seed=1).close()  # warm (module load, pool growth)
            best = None
            for _ in range(a.reps):
                torch.cuda.synchronize()
                c = Collection(off_d, tids_d, w.m, seed=1)
                st, inf = c.stats(), c.info()
                c.close()
                if best is None or st["build_ms"] < best[0]["build_ms"]:
                    best = (st, inf)
            st, inf = best
            line = dict(config=name, variant=var, nnz=w.nnz, build_ms=st["build_ms"],
                        k1_insert_ms=st["k1_insert_ms"], k1_encode_ms=st["k1_encode_ms"],
                        build_pre_ms=st["build_pre_ms"], build_post_ms=st["build_post_ms"],
                        launches=st["launches_build"], failures=inf["n_failures"],
                        arena_MB=inf["arena_bytes"] / 1e6,
                        insertions_per_s=2 * w.nnz / (st["k1_insert_ms"] / 1e3))
            if a.check:
                if ref is None:
                    ref = _reference(w)
                with Collection(off_d, tids_d, w.m, seed=1) as c:
                    got = c.pair_supports(threshold=w.threshold).cpu().numpy().astype(np.uint32).reshape(-1, 3)
                line["exact"] = bool(np.array_equal(got, ref[0]))
                line["checked_against"] = ref[1]
            print(json.dumps(line), flush=True)
        for k in ENV.values():
            os.environ.pop(k, None)


if __name__ == "__main__":
    main()
