"""NEXT-4 measurement: frequent triples end to end on the device (readings #26-#32).

Per config: frequent pairs (batmap_build + batmap_pair_supports), Apriori candidates
(batmap_candidate_triples), 3-of-4 BatMaps (batmap3_build) and the triple kernel
(batmap3_triple_supports) -- each timed with CUDA events (best of `reps`), the triple kernel's
work in word-triples (sum over candidates of the widest BatMap's words, r words for 4r bytes)
and its rate, and parity against the horizontal triple oracle (oracle/triples.c).

    python tools/triples_bench.py [--reps 3] [--thr C1=2] C3 C1
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1102_1003_b200 import Collection, Collection3, candidate_triples  # noqa: E402
from workloads import make_config  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    return out, a.elapsed_time(b)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--thr", nargs="*", default=["C1=2"])
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("configs", nargs="*", default=["C3", "C1"])
    a = ap.parse_args()
    thr_over = dict(kv.split("=") for kv in a.thr)
    for name in a.configs:
        w = make_config(name)
        thr = int(thr_over.get(name, w.threshold))
        off = torch.as_tensor(w.offsets).cuda()
        tids = torch.as_tensor(w.tids).cuda()
        best = {}
        for _ in range(a.reps + 1):
            c2, t_build2 = timed(lambda: Collection(off, tids, w.m, seed=1))
            pairs, t_pairs = timed(lambda: c2.pair_supports(threshold=thr))
            c2.close()
            cand, t_cand = timed(lambda: candidate_triples(pairs, w.n))
            c3, t_build3 = timed(lambda: Collection3(off, tids, w.m, seed=1))
            quads, t_tri = timed(lambda: c3.triple_supports(cand, threshold=thr))
            info = c3.info()
            c3.close()
            cur = dict(build2_ms=t_build2, pairs_ms=t_pairs, cand_ms=t_cand, build3_ms=t_build3, triples_ms=t_tri,
                       triples_kernel_ms=info["triples_ms"])
            for k, v in cur.items():
                best[k] = min(best.get(k, 1e30), v)
        lens = np.diff(w.offsets)
        s3 = info["s_shift"]
        r = np.maximum(np.maximum(2 ** np.ceil(np.log2(np.maximum(2 * lens, 1))).astype(np.int64), 2 ** s3), 128)
        cn = cand.cpu().numpy()
        word_triples = int(np.maximum(np.maximum(r[cn[:, 0]], r[cn[:, 1]]), r[cn[:, 2]]).sum()) if len(cn) else 0
        got = quads.cpu().numpy().astype(np.uint32)
        line = dict(config=name, n=w.n, m=w.m, threshold=thr, frequent_pairs=int(pairs.shape[0]),
                    candidates=int(cand.shape[0]), frequent_triples=int(got.shape[0]),
                    arena3_MB=info["arena_bytes"] / 1e6, failures3=info["n_failures"], **best,
                    word_triples=word_triples,
                    word_triples_per_s=word_triples / (best["triples_kernel_ms"] / 1e3) if word_triples else None,
                    l2_GBps=12.0 * word_triples / (best["triples_kernel_ms"] / 1e3) / 1e9 if word_triples else None,
                    step_ms=sum(best[k] for k in ("build2_ms", "pairs_ms", "cand_ms", "build3_ms", "triples_ms")))
        if not a.no_oracle:
            import oracle

            t0 = time.time()
            ref = oracle.triples_horizontal(w.offsets, w.tids, w.m, threshold=thr)
            line["oracle_s"] = round(time.time() - t0, 2)
            line["oracle_threads"] = oracle.num_threads()
            line["exact"] = bool(np.array_equal(got, ref))
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
