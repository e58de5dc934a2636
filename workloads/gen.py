"""Seeded generators of vertical tidlists (CSR) for the five BASELINE.json configs.

Vertical format: for item i the sorted set S_i of transaction ids, here
0-based in [0, m).  CSR: ``offsets`` int64[n+1], ``tids`` int32[nnz], each segment
strictly increasing.

* ``uniform`` -- the paper's generator ("for each transaction, including
  each of the n distinct items with probability p"), with m fixed instead of the
  total size.  Drawn per item as a Bernoulli(p) process over [0, m) via geometric
  gaps, which is equal in law to per-(item, transaction) Bernoulli inclusion.
* ``zipf`` -- kosarak-shaped skew: p_k = min(cap, c k^-alpha) with
  c solved so that sum_k p_k = avg items/transaction; ranks randomly permuted onto ids.
* ``quest`` -- Agrawal-Srikant style T40I10D100K-shaped data (the
  paper only names the dataset and its 4% density).

Everything is deterministic in ``seed`` (numpy PCG64).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = ["Workload", "uniform", "zipf", "quest", "to_horizontal", "make_config", "CONFIGS", "fimi_text"]


@dataclasses.dataclass
class Workload:
    name: str
    offsets: np.ndarray  # int64[n+1]
    tids: np.ndarray  # int32[nnz]
    m: int  # number of transactions
    threshold: int  # support threshold s
    meta: dict

    @property
    def n(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.tids.shape[0])


def _bernoulli_rows(rng: np.random.Generator, p: float, m: int, rows: int) -> list[np.ndarray]:
    """`rows` independent Bernoulli(p) subsets of [0, m), each sorted, via geometric gaps."""
    if p <= 0.0 or m == 0:
        return [np.empty(0, np.int32) for _ in range(rows)]
    if p >= 1.0:
        return [np.arange(m, dtype=np.int32) for _ in range(rows)]
    mean = m * p
    g = int(math.ceil(mean + 8.0 * math.sqrt(mean * (1.0 - p)) + 32))
    out: list[np.ndarray] = []
    chunk = max(1, min(rows, int(4e7 // max(g, 1))))
    done = 0
    while done < rows:
        c = min(chunk, rows - done)
        gaps = rng.geometric(p, size=(c, g)).astype(np.int64)
        pos = np.cumsum(gaps, axis=1) - 1
        for r in range(c):
            row = pos[r]
            while row[-1] < m:  # rare: not enough gaps drawn; extend this row
                more = np.cumsum(rng.geometric(p, size=g).astype(np.int64)) + row[-1]
                row = np.concatenate([row, more])
            out.append(row[row < m].astype(np.int32))
        done += c
    return out


def _csr(rows: list[np.ndarray]) -> tuple[np.ndarray, np.ndarray]:
    sizes = np.fromiter((len(r) for r in rows), dtype=np.int64, count=len(rows))
    offsets = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    tids = np.concatenate(rows).astype(np.int32) if rows else np.empty(0, np.int32)
    return offsets, tids


def uniform(n: int, m: int, p: float, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """n items, each in every one of m transactions independently with probability p."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return _csr(_bernoulli_rows(rng, p, m, n))


def zipf_probs(n: int, alpha: float = 1.0, cap: float = 0.6, avg: float = 8.1) -> np.ndarray:
    """p_k = min(cap, c k^-alpha), k = 1..n, with c chosen by bisection so sum p_k = avg."""
    k = np.arange(1, n + 1, dtype=np.float64)
    lo, hi = 0.0, float(avg) * 10.0 + 1.0
    for _ in range(200):
        c = 0.5 * (lo + hi)
        s = np.minimum(cap, c * k ** (-alpha)).sum()
        if s < avg:
            lo = c
        else:
            hi = c
    return np.minimum(cap, 0.5 * (lo + hi) * k ** (-alpha))


def zipf(n: int, m: int, seed: int, alpha: float = 1.0, cap: float = 0.6,
         avg: float = 8.1) -> tuple[np.ndarray, np.ndarray]:
    """Zipf-skewed tidlist lengths (kosarak-shaped); popularity ranks permuted onto ids."""
    rng = np.random.Generator(np.random.PCG64(seed))
    pk = zipf_probs(n, alpha, cap, avg)
    perm = rng.permutation(n)  # rank k -> item id perm[k]
    p_item = np.empty(n, dtype=np.float64)
    p_item[perm] = pk
    rows = []
    for i in range(n):
        rows.extend(_bernoulli_rows(rng, float(p_item[i]), m, 1))
    return _csr(rows)


def quest(D: int = 100_000, T: float = 40.0, I: float = 10.0, L: int = 2000, N: int = 1000,
          corr: float = 0.5, seed: int = 3) -> tuple[np.ndarray, np.ndarray]:
    """Agrawal-Srikant style generator (T40I10D100K shape), returned in vertical form.

    L potential patterns, sizes ~ Poisson(I) (>= 1); each pattern takes an Exp(corr)
    fraction of its items from the previous pattern, the rest uniformly.  Pattern
    weights ~ Exp(1) (normalised), corruption levels ~ N(0.5, 0.1) clipped to [0, 1].
    Transaction sizes ~ Poisson(T) (>= 1); a transaction is filled with weighted
    patterns, each corrupted by dropping random items while U(0,1) < its corruption
    level; a pattern that overflows the transaction is kept with probability 0.5,
    otherwise carried over to the next transaction.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    sizes = np.maximum(1, rng.poisson(I, size=L))
    patterns: list[np.ndarray] = []
    prev = np.empty(0, dtype=np.int64)
    for k in range(L):
        sz = int(sizes[k])
        frac = min(1.0, rng.exponential(corr)) if k > 0 else 0.0
        n_from_prev = min(len(prev), int(round(frac * sz)))
        take = rng.choice(prev, size=n_from_prev, replace=False) if n_from_prev > 0 else np.empty(0, np.int64)
        rest = rng.integers(0, N, size=sz * 2 + 4)
        items = list(dict.fromkeys(list(take.tolist()) + rest.tolist()))[:sz]
        pat = np.array(sorted(items), dtype=np.int64)
        patterns.append(pat)
        prev = pat
    weights = rng.exponential(1.0, size=L)
    weights /= weights.sum()
    cumw = np.cumsum(weights)
    corrupt = np.clip(rng.normal(0.5, 0.1, size=L), 0.0, 1.0)
    tsizes = np.maximum(1, rng.poisson(T, size=D))
    # pre-draw a generous stream of pattern picks
    picks = np.searchsorted(cumw, rng.random(size=int(D * (T / max(I, 1.0)) * 3) + 1024))
    picks = np.minimum(picks, L - 1)
    pi = 0
    carry: np.ndarray | None = None
    trans_items: list[np.ndarray] = []
    for b in range(D):
        target = int(tsizes[b])
        cur: set[int] = set()
        while len(cur) < target:
            if carry is not None:
                pat, carry = carry, None
            else:
                if pi >= len(picks):
                    picks = np.minimum(np.searchsorted(cumw, rng.random(size=len(picks))), L - 1)
                    pi = 0
                j = int(picks[pi])
                pi += 1
                pat = patterns[j]
                c = corrupt[j]
                if len(pat) > 0:
                    keep = np.ones(len(pat), dtype=bool)
                    while keep.any() and rng.random() < c:
                        idx = np.flatnonzero(keep)
                        keep[idx[rng.integers(0, len(idx))]] = False
                    pat = pat[keep]
            if len(cur) + len(pat) > target and len(cur) > 0:
                if rng.random() < 0.5:
                    cur.update(pat.tolist())
                else:
                    carry = pat
                break
            cur.update(pat.tolist())
        trans_items.append(np.array(sorted(cur), dtype=np.int64))
    # transpose horizontal -> vertical
    lens = np.fromiter((len(t) for t in trans_items), dtype=np.int64, count=D)
    flat_items = np.concatenate(trans_items) if D else np.empty(0, np.int64)
    flat_tids = np.repeat(np.arange(D, dtype=np.int64), lens)
    order = np.lexsort((flat_tids, flat_items))
    flat_items, flat_tids = flat_items[order], flat_tids[order]
    counts = np.bincount(flat_items, minlength=N).astype(np.int64)
    offsets = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return offsets, flat_tids.astype(np.int32)


def to_horizontal(offsets: np.ndarray, tids: np.ndarray, m: int) -> tuple[np.ndarray, np.ndarray]:
    """Transpose vertical CSR to horizontal CSR (transactions -> sorted item ids)."""
    n = offsets.shape[0] - 1
    items = np.repeat(np.arange(n, dtype=np.int64), np.diff(offsets))
    order = np.lexsort((items, tids.astype(np.int64)))
    t_sorted = tids.astype(np.int64)[order]
    i_sorted = items[order]
    counts = np.bincount(t_sorted, minlength=m).astype(np.int64)
    toff = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=toff[1:])
    return toff, i_sorted.astype(np.int32)


# BASELINE.json configs, concretised per SURVEY §8(d).
CONFIGS = {
    "C1": dict(kind="uniform", n=1000, m=10_000, p=0.01, threshold=5, seed=1),
    "C2": dict(kind="uniform", n=10_000, m=100_000, p=0.01, threshold=20, seed=2),
    "C3": dict(kind="quest", n=1000, m=100_000, threshold=500, seed=3),
    "C4": dict(kind="zipf", n=100_000, m=1_000_000, threshold=100, seed=4),
}
_C5_P = [0.001, 0.002, 0.005, 0.01, 0.02, 0.05, 0.10]
for _k, _p in enumerate(_C5_P):
    _m = 200_000
    _mu = _m * _p * _p
    _thr = max(2, int(math.ceil(_mu + 5.0 * math.sqrt(_mu))))
    CONFIGS[f"C5_p{_p:g}"] = dict(kind="uniform", n=20_000, m=_m, p=_p, threshold=_thr, seed=50 + _k)


def make_config(name: str, scale_items: float = 1.0, seed: int | None = None) -> Workload:
    """Instantiate a named config.  ``scale_items`` < 1 shrinks n (test-size variants)."""
    cfg = dict(CONFIGS[name])
    if seed is not None:
        cfg["seed"] = seed
    n = max(2, int(round(cfg["n"] * scale_items)))
    m = cfg["m"]
    if cfg["kind"] == "uniform":
        off, tids = uniform(n, m, cfg["p"], cfg["seed"])
    elif cfg["kind"] == "zipf":
        off, tids = zipf(n, m, cfg["seed"])
    elif cfg["kind"] == "quest":
        off, tids = quest(D=m, N=n, seed=cfg["seed"])
    else:  # pragma: no cover
        raise ValueError(cfg["kind"])
    return Workload(name=name, offsets=off, tids=tids, m=m, threshold=cfg["threshold"],
                    meta=dict(cfg, n=n))


def fimi_text(offsets: np.ndarray, tids: np.ndarray, m: int, *, labels: np.ndarray | None = None, seed: int = 0,
              messy: bool = False, final_newline: bool = True) -> bytes:
    """Write a vertical CSR as FIMI-repository text (one transaction per line, item labels
    separated by whitespace).  ``labels[i]`` is item i's label (default: i).
    ``messy`` varies the formatting the way real files do (tabs, runs of spaces, CRLF line
    ends, leading/trailing blanks, items repeated within a line, unsorted lines); every
    transaction -- empty ones too -- is one line."""
    toff, items = to_horizontal(offsets, tids, m)
    lab = np.arange(offsets.shape[0] - 1, dtype=np.int64) if labels is None else np.asarray(labels, np.int64)
    rng = np.random.default_rng(seed)
    if not messy:
        lines = [" ".join(map(str, lab[items[toff[t]:toff[t + 1]]].tolist())) for t in range(m)]
        body = "\n".join(lines)
        return (body + ("\n" if final_newline and m else "")).encode()
    seps = [" ", "  ", "\t", " \t ", "   "]
    out = []
    for t in range(m):
        row = lab[items[toff[t]:toff[t + 1]]].tolist()
        if row and rng.random() < 0.3:
            row = row + [row[int(rng.integers(len(row)))]]  # a repeated item
        rng.shuffle(row)
        s = (" " if rng.random() < 0.2 else "")
        s += "".join(str(v) + seps[int(rng.integers(len(seps)))] if k + 1 < len(row) else str(v)
                     for k, v in enumerate(row))
        s += (" " if rng.random() < 0.2 else "") + ("\r" if rng.random() < 0.3 else "")
        out.append(s)
    body = "\n".join(out)
    return (body + ("\n" if final_newline and m else "")).encode()
