"""oracle/batmap_ref.py -- TEST INFRASTRUCTURE ONLY.

The BatMap method of PAPER.md followed step by step, in the paper's order and
notation, in plain Python/numpy.  It exists to give the CUDA path *internal* parity
targets (the bytes the build writes, the raw counts the intersection produces); the
*output* parity target is the definition in ``pairs.c``.  It is pinned in
tests/test_oracle_batmap.py against the paper's worked example, the
paper's Fig. 5 assignments, a per-byte check of the SWAR closed form, the build
invariants of §2 and -- end to end -- against |S_i ∩ S_j| by sorted merge.

Readings of the paper (DESIGN.md §3 lists all of them; numbers follow SURVEY §8(c5)):
  #1  ⊥ is the byte 0x7F: codes are restricted to [0,126] by U = 127·2^s.
  #2  transactions are 0-based ids in [0, m); s = min{s : 127·2^s >= m}.
  #3  π_t is a seeded 4-round multiply/xorshift mixer mod 2^w, w = s+7,
      cycle-walked into [0, U); a caller-given table may replace it (test hook).
  #4  r_i = max(2^ceil(log2(2|S_i|)), 2^s, r_min).
  #5  |B_0| = 3 r_0 with r_0 = min_i r_i over the collection (caption P:407).
  #6  indicator b = 1 on the copy whose partner sits in the cyclically preceding
      table, order 1->2->3->1 (Fig. 5).
  #8  MaxLoop counts rounds of 3 swaps; default 16 + ceil(3 log2 r).
  #9  on a failed insertion of x: delete every occurrence of x, record (i, x) as
      failed, re-insert the nestless element once unless it is x; cascades repeat.
  #10 elements are inserted in ascending tid order.
  #11 corrections use set semantics per (pair, transaction).
  #17 4 entries per 32-bit word, entry e in byte lane e & 3 (little-endian).
  #18 entry e of the wider BatMap is compared with entry e mod 3 r_i of the narrower.
"""
from __future__ import annotations

import math

import numpy as np

NULL = 0x7F  # reading #1
M80 = 0x80808080
L01 = 0x01010101
MASK64 = (1 << 64) - 1


# ----------------------------------------------------------------------------- params
def derive_params(m: int) -> tuple[int, int]:
    """(s, U): smallest s with 127·2^s >= m ("log(m+1) - s <= 7", reading #2)."""
    s = 0
    while 127 * (1 << s) < m:
        s += 1
    return s, 127 * (1 << s)


def table_range(size: int, s: int, r_min: int) -> int:
    """r_i: power of two, ~2|S_i|, >= 2^s, >= r_min (reading #4)."""
    r = 1
    while r < 2 * size:
        r <<= 1
    return max(r, 1 << s, r_min)


def default_max_loop(r: int) -> int:
    """MaxLoop rounds (value unstated -> reading #8)."""
    return 16 + int(math.ceil(3 * math.log2(r)))


# ----------------------------------------------------------------------------- π_t
def splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def pi_keys(seed: int, s: int) -> list[list[int]]:
    """Round keys k_{t,r}, t = 0..2 (table t+1), r = 0..3: odd, reduced mod 2^w."""
    w = s + 7
    mask = (1 << w) - 1
    keys = []
    for t in range(3):
        row = []
        for r in range(4):
            z = splitmix64((seed + (4 * t + r) * 0x9E3779B97F4A7C15) & MASK64)
            row.append(((z & 0xFFFFFFFF) | 1) & mask)
        keys.append(row)
    return keys


def pi_table(seed: int, s: int) -> np.ndarray:
    """π_t(x) for t = 1..3 (rows 0..2) and all x in [0, U): permutations of [0, U).

    mix_t(v): 4 rounds of {v <- v·k_{t,r} mod 2^w; v <- v xor (v >> ceil(w/2))};
    π_t(x) = mix_t applied until the value is < U (cycle walking, reading #3).
    """
    U = 127 * (1 << s)
    w = s + 7
    mask = np.uint64((1 << w) - 1)
    half = np.uint64((w + 1) // 2)
    keys = pi_keys(seed, s)
    out = np.empty((3, U), dtype=np.int64)
    x = np.arange(U, dtype=np.uint64)
    for t in range(3):
        def mix(v):
            for r in range(4):
                v = (v * np.uint64(keys[t][r])) & mask
                v = v ^ (v >> half)
            return v
        v = mix(x.copy())
        bad = v >= U
        while bad.any():
            v[bad] = mix(v[bad])
            bad = v >= U
        out[t] = v.astype(np.int64)
    return out


# ----------------------------------------------------------------------------- layout
def h(t: int, v: int, r: int, r0: int) -> int:
    """h_t^(i) = |B_0|·floor((v mod r_i)/r_0) + (v mod r_0) + (t-1) r_0, |B_0| = 3 r_0."""
    return 3 * r0 * ((v % r) // r0) + (v % r0) + (t - 1) * r0


def table_of(q: int, r0: int) -> int:
    """Which hash table t in {1,2,3} the entry q belongs to under the superblock layout."""
    return (q % (3 * r0)) // r0 + 1


def pred(t: int) -> int:
    """Cyclic predecessor in the order 1 -> 2 -> 3 -> 1."""
    return 3 if t == 1 else t - 1


def indicator(t_self: int, t_other: int) -> int:
    """b for the copy in table t_self when the partner is in t_other (Fig. 5, reading #6)."""
    if t_self == t_other:
        raise ValueError("two copies never share a table")
    return 1 if t_other == pred(t_self) else 0


def encode_entry(code: int, b: int) -> int:
    """8-bit entry: indicator as MSB, 7 MSBs of π_t(x) below it."""
    if not 0 <= code <= 126:
        raise ValueError("code 127 is reserved for ⊥")
    return (b << 7) | code


# ----------------------------------------------------------------------------- build
class BatMap:
    """One set's BatMap A^(i) built with the generalized cuckoo INSERT."""

    def __init__(self, S, r: int, r0: int, pi, s: int, max_loop: int | None = None):
        self.S = [int(x) for x in S]
        self.r, self.r0, self.s = r, r0, s
        self.pi = pi  # pi[t-1][x] = π_t(x)
        self.max_loop = default_max_loop(r) if max_loop is None else max_loop
        self.A: list[int | None] = [None] * (3 * r)  # None = ⊥
        self.failed: list[int] = []
        self.moves = 0

    def pos(self, t: int, x: int) -> int:
        return h(t, int(self.pi[t - 1][x]), self.r, self.r0)

    def insert(self, tau: int) -> int | None:
        """INSERT(τ) of P:293-303: swap τ into A_1, A_2, A_3 cyclically, MaxLoop rounds."""
        A = self.A
        for _ in range(self.max_loop):
            for t in (1, 2, 3):
                p = self.pos(t, tau)
                tau, A[p] = A[p], tau
                self.moves += 1
                if tau is None:
                    return None
        return tau

    def delete(self, x: int) -> None:
        for t in (1, 2, 3):
            p = self.pos(t, x)
            if self.A[p] == x:
                self.A[p] = None

    def build(self) -> "BatMap":
        """Two insertions per element; failures per P:310 and reading #9."""
        for x in sorted(self.S):  # reading #10
            y = self.insert(x)
            if y is None:
                y = self.insert(x)
            if y is None:
                continue
            cur, nest = x, y
            while True:
                self.delete(cur)
                self.failed.append(cur)
                if nest == cur:
                    break
                z = self.insert(nest)
                if z is None:
                    break
                cur, nest = nest, z
        return self

    def copies(self, x: int) -> list[int]:
        return [t for t in (1, 2, 3) if self.A[self.pos(t, x)] == x]

    def encode(self) -> np.ndarray:
        """Entry bytes in order e = 0..3r-1; ⊥ -> 0x7F."""
        out = np.full(3 * self.r, NULL, dtype=np.uint8)
        for q, x in enumerate(self.A):
            if x is None:
                continue
            t = table_of(q, self.r0)
            others = [u for u in self.copies(x) if u != t]
            assert len(others) == 1, "every stored element has exactly two copies"
            code = int(self.pi[t - 1][x]) >> self.s
            out[q] = encode_entry(code, indicator(t, others[0]))
        return out

    @property
    def live(self) -> int:
        return len(self.S) - len(self.failed)


def words(entries: np.ndarray) -> np.ndarray:
    """Pack entry bytes 4 per little-endian uint32 word (reading #17)."""
    return np.frombuffer(np.ascontiguousarray(entries, dtype=np.uint8).tobytes(), dtype="<u4").copy()


# ----------------------------------------------------------------------------- compare
def swar_count(x: int, y: int) -> int:
    """The paper's branch-free count of matches between two words, literally."""
    p = (((x ^ y) | 0x80808080) - 0x01010101) & 0xFFFFFFFF
    pp = (p ^ 0xFFFFFFFF) & ((x | y) & 0x80808080)
    return ((pp >> 7) + (pp >> 15) + (pp >> 23) + (pp >> 31)) & 7


def swar_count_np(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Vectorised form of swar_count over uint32 arrays (same formulas)."""
    x = x.astype(np.uint64)
    y = y.astype(np.uint64)
    p = (((x ^ y) | 0x80808080) - 0x01010101) & 0xFFFFFFFF
    pp = (p ^ 0xFFFFFFFF) & ((x | y) & 0x80808080)
    return (((pp >> 7) + (pp >> 15) + (pp >> 23) + (pp >> 31)) & 7).astype(np.int64)


def count_pair(Bi: np.ndarray, Bj: np.ndarray) -> int:
    """|stored(B_i) ∩ stored(B_j)| by word-wise comparison with wrap-around (#18).

    Bi, Bj are word arrays (3r/4 words each).  Each word of the wider BatMap is compared
    with word (w mod W_narrow) of the narrower one.
    """
    if len(Bi) > len(Bj):
        Bi, Bj = Bj, Bi
    Wi, Wj = len(Bi), len(Bj)
    if Wi == 0:
        return 0
    idx = np.arange(Wj) % Wi
    return int(swar_count_np(Bj, Bi[idx]).sum())


# ----------------------------------------------------------------------------- pipeline
class Collection:
    """All BatMaps of an instance sharing π, s and r_0."""

    def __init__(self, offsets, tids, m: int, seed: int = 0, r_min: int = 128,
                 max_loop: int | None = None, pi: np.ndarray | None = None):
        offsets = np.asarray(offsets, dtype=np.int64)
        tids = np.asarray(tids, dtype=np.int64)
        self.n = offsets.shape[0] - 1
        self.m = m
        self.s, self.U = derive_params(m)
        self.pi = pi_table(seed, self.s) if pi is None else np.asarray(pi, dtype=np.int64)
        self.sets = [tids[offsets[i]:offsets[i + 1]] for i in range(self.n)]
        self.r = [table_range(len(S), self.s, r_min) for S in self.sets]
        self.r0 = min(self.r) if self.r else r_min  # reading #5
        pil = [self.pi[t].tolist() for t in range(3)]
        self.maps = [BatMap(S, self.r[i], self.r0, pil, self.s, max_loop).build()
                     for i, S in enumerate(self.sets)]
        self.bytes = [bm.encode() for bm in self.maps]
        self.words = [words(b) for b in self.bytes]
        # sort by increasing width; stable by id (reading #16)
        self.order = sorted(range(self.n), key=lambda i: (self.r[i], i))

    def failures(self) -> list[tuple[int, int]]:
        """F as (item, tid) pairs (F_b = items whose insertion of b failed)."""
        return sorted((i, int(x)) for i, bm in enumerate(self.maps) for x in bm.failed)

    def raw_count(self, i: int, j: int) -> int:
        return count_pair(self.words[i], self.words[j])

    def corrections(self) -> dict[tuple[int, int], int]:
        """|M| per pair: pairs (min(a,c), max(a,c)) for a in F_b, c in A_b, as a set
        of (pair, b) triples (reading #11)."""
        Fb: dict[int, set[int]] = {}
        for i, bm in enumerate(self.maps):
            for b in bm.failed:
                Fb.setdefault(int(b), set()).add(i)
        Ab: dict[int, list[int]] = {b: [] for b in Fb}
        for i, S in enumerate(self.sets):
            for b in S.tolist():
                if b in Ab:
                    Ab[b].append(i)
        M: set[tuple[int, int, int]] = set()
        for b, fa in Fb.items():
            for a in fa:
                for c in Ab[b]:
                    if c != a:
                        M.add((min(a, c), max(a, c), b))
        corr: dict[tuple[int, int], int] = {}
        for a, c, _b in M:
            corr[(a, c)] = corr.get((a, c), 0) + 1
        return corr

    def pair_supports(self, items=None, threshold: int = 1) -> np.ndarray:
        """Triples (i, j, supp), i<j caller ids, supp = raw count + |M_{ij}| >= threshold."""
        sel = sorted(set(range(self.n) if items is None else (int(x) for x in items)))
        corr = self.corrections()
        out = []
        for u, i in enumerate(sel):
            for j in sel[u + 1:]:
                s = self.raw_count(i, j) + corr.get((i, j), 0)
                if s >= threshold:
                    out.append((i, j, s))
        return np.array(out, dtype=np.uint32).reshape(-1, 3)
