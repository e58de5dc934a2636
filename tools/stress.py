"""Randomized exactness stress of the whole path against the oracle, for a fixed wall-clock budget:
random shapes (uniform or Zipf tidlists, a few long items to reach the cluster and global build
tiers), forced insertion failures, item subsets, both K1 cluster policies, the byte-table K1 tier
(never / default / every class), both K2 tile widths, K2's balanced mode on and off, the byte tier's staged pack, and -- where horizontal triple counting is
cheap -- the NEXT-4 triples path (candidates from the frequent pairs, 3-of-4 BatMaps, supports).
The concurrent build is timing-dependent (reading #9b), so rare interleavings only show up over
many runs; every run must be bit-exact.  (K1 side stream on/off too.)

    python tools/stress.py [seconds]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def case(rng):
    from workloads import uniform, zipf

    m = int(rng.choice([300, 2000, 20000, 100000, 300000]))
    n = int(rng.integers(2, 900))
    if rng.random() < 0.5:
        off, tids = uniform(n, m, float(rng.choice([0.002, 0.01, 0.05])), int(rng.integers(1 << 30)))
    else:
        off, tids = zipf(n, m, int(rng.integers(1 << 30)))
    rows = [tids[off[i]:off[i + 1]] for i in range(len(off) - 1)]
    for _ in range(int(rng.integers(0, 3))):  # long items: cluster / global build tiers
        size = int(min(m // 2, rng.choice([3000, 9000, 20000, 70000])))
        if size > 0:
            rows.append(np.sort(rng.choice(m, size=size, replace=False)).astype(np.int32))
    o = np.zeros(len(rows) + 1, np.int64)
    o[1:] = np.cumsum([len(r) for r in rows])
    return o, (np.concatenate(rows) if rows else np.zeros(0, np.int32)).astype(np.int32), m


def main():
    import torch

    import oracle
    from paper_1102_1003_b200 import Collection, Collection3, candidate_triples

    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    rng = np.random.default_rng(int(os.environ.get("STRESS_SEED", "12345")))
    t0 = time.time()
    runs = 0
    tri_runs = 0
    while time.time() - t0 < budget:
        off, tids, m = case(rng)
        n = len(off) - 1
        os.environ["BATMAP_K1_SPREAD"] = str(int(rng.integers(0, 2)))
        os.environ["BATMAP_K2_TN"] = str(int(rng.choice([64, 128])))
        os.environ["BATMAP_K1_SIDE"] = str(int(rng.integers(0, 2)))
        os.environ["BATMAP_K2_BALANCE"] = str(int(rng.integers(0, 2)))
        os.environ["BATMAP_K1_STAGE"] = str(rng.choice(["0", "1", "4"]))  # byte-tier staged pack
        byte = str(rng.choice(["", "0", "all"]))
        if byte:
            os.environ["BATMAP_K1_BYTE"] = byte
        else:
            os.environ.pop("BATMAP_K1_BYTE", None)
        max_loop = int(rng.choice([0, 0, 1, 2]))
        thr = int(rng.choice([1, 2, 3, 10]))
        items = None
        if rng.random() < 0.3 and n > 2:
            items = np.sort(rng.choice(n, size=int(rng.integers(2, n + 1)), replace=False)).astype(np.int32)
        ref = oracle.pairs_horizontal(off, tids, m, items=items, threshold=thr)
        with Collection(torch.as_tensor(off).cuda(), torch.as_tensor(tids).cuda(), m,
                        seed=int(rng.integers(1 << 30)), max_loop=max_loop) as c:
            sel = None if items is None else torch.as_tensor(items).cuda()
            got = c.pair_supports(sel, threshold=thr).cpu().numpy().astype(np.uint32)
            nf = c.info()["n_failures"]
        if not np.array_equal(got, ref):
            print(f"MISMATCH run {runs}: n={n} m={m} max_loop={max_loop} thr={thr} items={items is not None} "
                  f"spread={os.environ['BATMAP_K1_SPREAD']} tn={os.environ['BATMAP_K2_TN']} byte={byte} failures={nf}")
            sys.exit(1)
        runs += 1
        lens = np.bincount(tids, minlength=m).astype(np.float64) if len(tids) else np.zeros(1)
        if items is None and float((lens ** 3).sum()) / 6 < 3e8:  # NEXT-4 where the oracle is cheap
            t_ref = oracle.triples_horizontal(off, tids, m, threshold=thr)
            o_d, t_d = torch.as_tensor(off).cuda(), torch.as_tensor(tids).cuda()
            cand = candidate_triples(torch.as_tensor(ref.astype(np.int32)).cuda(), n)
            with Collection3(o_d, t_d, m, seed=int(rng.integers(1 << 30)), max_loop=max_loop,
                             serial=bool(rng.random() < 0.1)) as c3:
                q = c3.triple_supports(cand, threshold=thr).cpu().numpy().astype(np.uint32)
            if not np.array_equal(q, t_ref):
                print(f"TRIPLES MISMATCH run {runs}: n={n} m={m} max_loop={max_loop} thr={thr} "
                      f"got {q.shape} ref {t_ref.shape}")
                sys.exit(1)
            tri_runs += 1
    print(f"stress ok: {runs} random runs bit-exact in {time.time() - t0:.0f} s ({tri_runs} with the triples path)")


if __name__ == "__main__":
    main()
