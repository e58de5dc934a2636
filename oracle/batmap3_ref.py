"""oracle/batmap3_ref.py -- TEST INFRASTRUCTURE ONLY (NEXT-4).

3-of-4 BatMaps for itemsets of size 3, followed step by step in plain Python/numpy.  The paper
leaves larger itemsets open and sketches this route: "a generalization of batmaps
that store items in d out of d+1 places.  This would ensure that itemsets of size up to d would
have at least one position witnessing their intersection."  With d = 3 every element of S_i is
stored in three of four tables, so any three sets sharing x all store x in at least one common
table.  Counting each common element exactly once needs an entry-level rule the paper does not
give; the readings below (#26-#32) fix one, chosen as the generalisation of Fig. 5.
This module gives the CUDA path internal parity targets (the bytes the serial build writes, the
raw counts of the triple kernel); the OUTPUT parity target is the definition in triples.c.

Readings:
  #26 d = 3: four tables t = 1..4 with permutations π_1..π_4, the mixer of reading #3 with the
      round keys k_{t,r} = splitmix64(seed + (4t + r)·φ) for t = 0..3.
  #27 6-bit codes: s3 = min{s : 63·2^s >= m}, U3 = 63·2^s3, code = π_t(x) >> s3 in [0, 62],
      ⊥ = code 63 (reading #1's argument with one bit less); r_i = max(2^ceil(log2 2|S_i|),
      2^s3, r_min) (P:421 with s3), r_0 = min r_i; superblocks of 4 r_0 (P:378 with four tables):
      h_t(x) = 4 r_0 floor((π_t(x) mod r_i)/r_0) + (t-1) r_0 + (π_t(x) mod r_0); 4 r_i bytes.
  #28 INSERT swaps through A_1, A_2, A_3, A_4 cyclically for MaxLoop rounds
      (default 16 + ceil(3 log2 r), reading #8) and is called THREE times per element (d = 3,
      P:629); a failed insertion deletes every copy of x, records (i, x) and re-inserts the
      nestless element unless it is x (reading #9); ascending tid order (reading #10).
  #29 entry byte = code | B1 << 6 | B2 << 7, with m = the (0-based) table that does NOT hold x:
      table 0: B1 = 1 (present); table 1: B1 = [m = 0]; tables 2, 3: B1 = [m = 0], B2 = [m = 1].
      ⊥ = 0x3F.
  #30 triple count: an element common to the three BatMaps is counted at the LOWEST table all
      three store it in: at an aligned position of table t whose three codes are equal (and not
      ⊥), count iff {0..t-1} ⊆ {m_i, m_j, m_k}:  t = 0: B1 of the first;  t = 1: any B1;
      t = 2: any B1 and any B2;  t = 3: any B1, any B2 and any N (N = not B1 and not B2, i.e.
      m = 2).  Wrap-around alignment as reading #18 (entry e of the wider <-> e mod 4 r of the
      narrower; the superblock layout puts aligned entries in the same table).
  #31 corrections with set semantics per (triple, transaction): supp = c + |{b in S_i ∩ S_j ∩
      S_k : (i,b) in F or (j,b) in F or (k,b) in F}| (P:469-474 generalised, reading #11).
  #32 candidates: triples i < j < k all of whose pairs are frequent (supp >= s); exact, since
      supp(i,j,k) <= supp of each of its pairs.
"""
from __future__ import annotations

import math

import numpy as np

from .batmap_ref import splitmix64

NULL3 = 0x3F
MASK64 = (1 << 64) - 1
T = 4  # tables (d + 1)
D = 3  # copies per element


def derive_params3(m: int) -> tuple[int, int]:
    """(s3, U3): smallest s with 63·2^s >= m (reading #27)."""
    s = 0
    while 63 * (1 << s) < m:
        s += 1
    return s, 63 * (1 << s)


def table_range3(size: int, s3: int, r_min: int) -> int:
    r = 1
    while r < 2 * size:
        r <<= 1
    return max(r, 1 << s3, r_min)


def default_max_loop(r: int) -> int:
    return 16 + int(math.ceil(3 * math.log2(r)))


def pi_keys4(seed: int, s3: int) -> list[list[int]]:
    w = s3 + 6
    mask = (1 << w) - 1
    keys = []
    for t in range(T):
        row = []
        for r in range(4):
            z = splitmix64((seed + (4 * t + r) * 0x9E3779B97F4A7C15) & MASK64)
            row.append(((z & 0xFFFFFFFF) | 1) & mask)
        keys.append(row)
    return keys


def pi_table4(seed: int, s3: int) -> np.ndarray:
    """π_t(x), t = 1..4 (rows 0..3), x in [0, U3): mixer on w = s3 + 6 bits, cycle-walked into [0, U3)."""
    U = 63 * (1 << s3)
    w = s3 + 6
    mask = np.uint64((1 << w) - 1)
    half = np.uint64((w + 1) // 2)
    keys = pi_keys4(seed, s3)
    out = np.empty((T, U), dtype=np.int64)
    x = np.arange(U, dtype=np.uint64)
    for t in range(T):
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


def h4(t: int, v: int, r: int, r0: int) -> int:
    """h_t = 4 r_0 floor((v mod r)/r_0) + (v mod r_0) + (t-1) r_0, t = 1..4 (reading #27)."""
    return 4 * r0 * ((v % r) // r0) + (v % r0) + (t - 1) * r0


def table_of4(q: int, r0: int) -> int:
    return (q % (4 * r0)) // r0 + 1


def encode_entry3(code: int, t: int, missing: int) -> int:
    """Entry byte of reading #29; t and missing are 1-based tables (missing = the table without x)."""
    if not 0 <= code <= 62:
        raise ValueError("code 63 is reserved for ⊥")
    if missing == t:
        raise ValueError("an entry's own table holds it")
    m = missing - 1
    if t == 1:
        return code | 0x40
    b1 = 1 if m == 0 else 0
    b2 = 1 if (m == 1 and t >= 3) else 0
    return code | (b1 << 6) | (b2 << 7)


class BatMap3:
    """One set's 3-of-4 BatMap built with INSERT called three times per element (reading #28)."""

    def __init__(self, S, r: int, r0: int, pi, s3: int, max_loop: int | None = None):
        self.S = [int(x) for x in S]
        self.r, self.r0, self.s3 = r, r0, s3
        self.pi = pi
        self.max_loop = default_max_loop(r) if max_loop is None else max_loop
        self.A: list[int | None] = [None] * (T * r)
        self.failed: list[int] = []

    def pos(self, t: int, x: int) -> int:
        return h4(t, int(self.pi[t - 1][x]), self.r, self.r0)

    def insert(self, tau: int) -> int | None:
        A = self.A
        for _ in range(self.max_loop):
            for t in (1, 2, 3, 4):
                p = self.pos(t, tau)
                tau, A[p] = A[p], tau
                if tau is None:
                    return None
        return tau

    def delete(self, x: int) -> None:
        for t in (1, 2, 3, 4):
            p = self.pos(t, x)
            if self.A[p] == x:
                self.A[p] = None

    def build(self) -> "BatMap3":
        for x in sorted(self.S):
            y = None
            for _ in range(D):
                y = self.insert(x)
                if y is not None:
                    break
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
        return [t for t in (1, 2, 3, 4) if self.A[self.pos(t, x)] == x]

    def encode(self) -> np.ndarray:
        out = np.full(T * self.r, NULL3, dtype=np.uint8)
        for q, x in enumerate(self.A):
            if x is None:
                continue
            t = table_of4(q, self.r0)
            have = self.copies(x)
            assert len(have) == D, "every stored element has exactly three copies"
            missing = ({1, 2, 3, 4} - set(have)).pop()
            out[q] = encode_entry3(int(self.pi[t - 1][x]) >> self.s3, t, missing)
        return out


def words(entries: np.ndarray) -> np.ndarray:
    return np.frombuffer(np.ascontiguousarray(entries, dtype=np.uint8).tobytes(), dtype="<u4").copy()


def entry_counts(a: int, b: int, c: int, t: int) -> bool:
    """Reading #30 on three aligned entry bytes of table t (1-based), per entry (plain form)."""
    ca, cb, cc = a & 0x3F, b & 0x3F, c & 0x3F
    if not (ca == cb == cc) or ca == 0x3F:
        return False
    if t == 1:
        return bool(a & 0x40)
    any1 = bool((a | b | c) & 0x40)
    any2 = bool((a | b | c) & 0x80)
    anyn = any(not (e & 0xC0) for e in (a, b, c))
    if t == 2:
        return any1
    if t == 3:
        return any1 and any2
    return any1 and any2 and anyn


def count_triple(Ei: np.ndarray, Ej: np.ndarray, Ek: np.ndarray, r0: int) -> int:
    """Raw count over entry bytes with wrap-around: entry e of the widest <-> e mod len of the others."""
    L = max(len(Ei), len(Ej), len(Ek))
    n = 0
    for e in range(L):
        t = table_of4(e, r0)
        if entry_counts(int(Ei[e % len(Ei)]), int(Ej[e % len(Ej)]), int(Ek[e % len(Ek)]), t):
            n += 1
    return n


class Collection3:
    """All 3-of-4 BatMaps of an instance (shared π, s3, r_0)."""

    def __init__(self, offsets, tids, m: int, seed: int = 0, r_min: int = 128, max_loop: int | None = None,
                 pi: np.ndarray | None = None):
        offsets = np.asarray(offsets, dtype=np.int64)
        tids = np.asarray(tids, dtype=np.int64)
        self.n = offsets.shape[0] - 1
        self.s3, self.U3 = derive_params3(m)
        self.pi = pi_table4(seed, self.s3) if pi is None else np.asarray(pi, dtype=np.int64)
        self.sets = [tids[offsets[i]:offsets[i + 1]] for i in range(self.n)]
        self.r = [table_range3(len(S), self.s3, r_min) for S in self.sets]
        self.r0 = min(self.r) if self.r else r_min
        pil = [self.pi[t].tolist() for t in range(T)]
        self.maps = [BatMap3(S, self.r[i], self.r0, pil, self.s3, max_loop).build() for i, S in enumerate(self.sets)]
        self.bytes = [bm.encode() for bm in self.maps]

    def failures(self) -> list[tuple[int, int]]:
        return sorted((i, int(x)) for i, bm in enumerate(self.maps) for x in bm.failed)

    def raw_count(self, i: int, j: int, k: int) -> int:
        return count_triple(self.bytes[i], self.bytes[j], self.bytes[k], self.r0)

    def correction(self, i: int, j: int, k: int) -> int:
        """|{b in S_i ∩ S_j ∩ S_k : b failed in i, j or k}| (reading #31)."""
        F = set(self.maps[i].failed) | set(self.maps[j].failed) | set(self.maps[k].failed)
        common = set(self.sets[i].tolist()) & set(self.sets[j].tolist()) & set(self.sets[k].tolist())
        return len(F & common)

    def triple_supports(self, triples) -> np.ndarray:
        out = []
        for i, j, k in triples:
            out.append(self.raw_count(i, j, k) + self.correction(i, j, k))
        return np.array(out, dtype=np.uint32)
