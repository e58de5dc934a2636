"""Load balance of the multi-GPU partition, measured on ONE GPU: every part p of an N-way run
(batmap_build_shard for the sharded build, batmap_pair_supports_part for the pair tiles) is run
in isolation and timed with the library's CUDA events.  With one rank per GPU the ranks run
these parts concurrently, so the N-GPU step is bounded below by the slowest part; the printed
`eff_bound` = T(N=1) / (N * max_p T_p) is the scaling efficiency the partition allows before
any communication (the BatMap all_gather and the triple gather).  Pair times are
the K2 + K3 kernel times (in a real run each rank's plan is prepared during its own build; here
one collection re-plans per part, which `pairs_ms` would include); every (config, N) is run once
untimed first (one-time module loading and pool growth).

    python tools/part_balance.py [C4 C2 C5_p0.01] [--parts 2 4 8]
"""
import argparse
import json
import os
import sys


sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C4", "C2", "C5_p0.01"])
    ap.add_argument("--parts", type=int, nargs="*", default=[2, 4, 8])
    a = ap.parse_args()
    import torch

    from paper_1102_1003_b200 import Collection
    from workloads import make_config

    for name in a.configs:
        w = make_config(name)
        off = torch.as_tensor(w.offsets).cuda()
        tids = torch.as_tensor(w.tids).cuda()
        Collection(off, tids, w.m, seed=1).close()  # warm-up build
        with Collection(off, tids, w.m, seed=1) as c:  # the N = 1 reference
            c.pair_supports(threshold=w.threshold)
            t1_build = c.stats()["build_ms"]
            c.pair_supports(threshold=w.threshold)
            st = c.stats()
            t1_pairs, k1 = st["k2_ms"] + st["k3_ms"], st["k2_ms"]
            K1 = st["n_results"]
            rows = []
            for N in a.parts:
                pairs, k2, wc, K = [], [], [], 0
                for p in range(N):
                    c.pair_supports(threshold=w.threshold, part=p, n_parts=N)  # warm
                for p in range(N):
                    got = c.pair_supports(threshold=w.threshold, part=p, n_parts=N)
                    s = c.stats()
                    pairs.append(s["k2_ms"] + s["k3_ms"])
                    k2.append(s["k2_ms"])
                    wc.append(s["word_compares"])
                    K += got.shape[0]
                builds = []
                Collection(off, tids, w.m, seed=1, part=N - 1, n_parts=N).close()  # warm
                for p in range(N):  # sharded build: part p builds 1/N of every width class
                    with Collection(off, tids, w.m, seed=1, part=p, n_parts=N) as cp:
                        builds.append(cp.stats()["build_ms"])
                rows.append({"N": N, "pairs_ms": pairs, "k2_ms": k2, "build_ms": builds,
                             "word_compares_max_over_mean": max(wc) / (sum(wc) / N),
                             "pairs_eff_bound": t1_pairs / (N * max(pairs)),
                             "k2_eff_bound": k1 / (N * max(k2)),
                             "build_eff_bound": t1_build / (N * max(builds)),
                             "step_eff_bound": (t1_pairs + t1_build) / (N * (max(pairs) + max(builds))),
                             "triples_equal_union": K == K1})
        print(json.dumps({"config": name, "n": w.n, "m": w.m, "N1": {"pairs_ms": t1_pairs, "build_ms": t1_build,
                                                                      "k2_ms": k1, "K": K1}, "parts": rows}),
              flush=True)


if __name__ == "__main__":
    main()
