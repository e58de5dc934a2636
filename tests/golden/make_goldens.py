"""Write the full-size C5 density-sweep goldens under tests/golden/c5/ -- ORACLE ONLY.

This script imports nothing but ``oracle/`` (the CPU definition oracle) and ``workloads/``
(the seeded generators, no method arithmetic); no value it stores comes from the CUDA path.

For every C5 density point (BASELINE.json configs[4]; P:536-543 density sweep, generator
P:503-504) it
  1. regenerates the seeded workload and records a SHA-256 of its CSR (so a test can prove
     it runs on the very input the golden was computed from);
  2. runs the horizontal pair-counting oracle (``oracle_pairs_horizontal``) over
     ALL C(20000, 2) pairs at a *low* threshold ``t_low`` -- the smallest threshold whose
     expected number of emitted pairs under the binomial model Bin(m, p^2) is <= 1.5e5, so
     the support distribution just above the official threshold is exercised -- and stores
     those triples; the official-threshold result is exactly the subset supp >= s;
  3. cross-checks with the second, independent oracle (sorted merge): every stored
     pair, plus random pairs whose merge support must be < t_low (i.e. correctly absent);
  4. writes ``<name>.npz`` (per-row counts of i, then j and supp) and ``manifest.json``.

Cached by (generator, params, seed): a point whose manifest entry matches is skipped unless
``--force``.  Usage::

    python tests/golden/make_goldens.py [--force] [--random-pairs N] [C5_p0.001 ...]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from workloads import CONFIGS, make_config  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "c5")

# smallest t with C(n,2) * P[Bin(m, p^2) >= t] <= 1.5e5 (capped at the official threshold);
# computed once with scipy.stats.binom.sf, a test-sizing choice only (no method arithmetic).
T_LOW = {"C5_p0.001": 3, "C5_p0.002": 6, "C5_p0.005": 14, "C5_p0.01": 37,
         "C5_p0.02": 111, "C5_p0.05": 573, "C5_p0.1": 2144}


def csr_sha256(offsets: np.ndarray, tids: np.ndarray) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(offsets, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(tids, dtype="<i4").tobytes())
    return h.hexdigest()


def triples_sha256(t: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(t, dtype="<u4").tobytes()).hexdigest()


def save_triples(path: str, t: np.ndarray, n: int) -> None:
    counts = np.bincount(t[:, 0].astype(np.int64), minlength=n).astype(np.uint32)
    np.savez_compressed(path, row_counts=counts, j=t[:, 1].astype(np.uint16 if n <= 65536 else np.uint32),
                        supp=t[:, 2].astype(np.uint32))


def load_triples(path: str) -> np.ndarray:
    """Inverse of save_triples: uint32 [K, 3] sorted by (i, j)."""
    z = np.load(path)
    counts = z["row_counts"].astype(np.int64)
    i = np.repeat(np.arange(counts.shape[0], dtype=np.uint32), counts)
    return np.stack([i, z["j"].astype(np.uint32), z["supp"].astype(np.uint32)], axis=1)


def make_one(name: str, n_random: int, manifest: dict, force: bool) -> dict:
    cfg = CONFIGS[name]
    key = dict(generator=cfg["kind"], n=cfg["n"], m=cfg["m"], p=cfg["p"], seed=cfg["seed"])
    old = manifest.get(name)
    if old and not force and old.get("key") == key and os.path.exists(os.path.join(OUT, old["file"])):
        print(f"{name}: cached", flush=True)
        return old
    t0 = time.time()
    w = make_config(name)
    gen_s = time.time() - t0
    t_low = T_LOW[name]
    assert t_low <= w.threshold
    t1 = time.time()
    got = oracle.pairs_horizontal(w.offsets, w.tids, w.m, threshold=t_low)
    horiz_s = time.time() - t1
    # second oracle on every stored pair (they must agree exactly) ...
    t2 = time.time()
    mc = oracle.merge_list(w.offsets, w.tids, got[:, 0], got[:, 1])
    assert np.array_equal(mc, got[:, 2]), f"{name}: merge and horizontal oracles disagree on emitted pairs"
    # ... and on random pairs: each is either emitted with the same support or below t_low
    rng = np.random.default_rng(12345)
    a = rng.integers(0, w.n, size=n_random)
    b = rng.integers(0, w.n, size=n_random)
    keep = a != b
    pi = np.minimum(a, b)[keep].astype(np.int32)
    pj = np.maximum(a, b)[keep].astype(np.int32)
    rs = oracle.merge_list(w.offsets, w.tids, pi, pj)
    key_got = got[:, 0].astype(np.int64) * w.n + got[:, 1]
    key_r = pi.astype(np.int64) * w.n + pj
    pos = np.searchsorted(key_got, key_r)
    hit = (pos < key_got.shape[0]) & (key_got[np.minimum(pos, key_got.shape[0] - 1)] == key_r)
    assert np.all(rs[~hit] < t_low), f"{name}: a random pair above t_low is missing from the horizontal output"
    assert np.array_equal(rs[hit], got[pos[hit], 2]), f"{name}: random-pair supports disagree"
    merge_s = time.time() - t2
    fname = f"{name}.npz"
    save_triples(os.path.join(OUT, fname), got, w.n)
    assert np.array_equal(load_triples(os.path.join(OUT, fname)), got)
    official = got[got[:, 2] >= w.threshold]
    ent = dict(key=key, file=fname, nnz=w.nnz, csr_sha256=csr_sha256(w.offsets, w.tids),
               threshold=w.threshold, t_low=t_low, K=int(official.shape[0]), K_low=int(got.shape[0]),
               sha256=triples_sha256(official), sha256_low=triples_sha256(got),
               max_support=int(got[:, 2].max()) if got.shape[0] else 0,
               merge_checked_pairs=int(got.shape[0] + pi.shape[0]),
               oracle="oracle_pairs_horizontal (all pairs) + oracle_merge_list (stored + random pairs)",
               threads=oracle.num_threads(), gen_s=round(gen_s, 1), horizontal_s=round(horiz_s, 1),
               merge_s=round(merge_s, 1))
    print(name, json.dumps(ent), flush=True)
    return ent


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*")
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--random-pairs", type=int, default=200_000)
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    mpath = os.path.join(OUT, "manifest.json")
    manifest = json.load(open(mpath)) if os.path.exists(mpath) else {}
    for name in a.names or list(T_LOW):
        manifest[name] = make_one(name, a.random_pairs, manifest, a.force)
        with open(mpath, "w") as f:
            json.dump(manifest, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
