"""oracle/ -- TEST INFRASTRUCTURE ONLY.

The plain, slow, obviously-correct CPU oracle for the BatMap hot path
(SURVEY.md §8(c)).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything under ``oracle/``.
The product path (``paper_1102_1003_b200``) never imports it, and this package never
imports the product: the two share no code, headers, tables or helpers.  Only the
seeded input generators in ``workloads/`` (no method arithmetic) serve both.

Contents
  pairs.c        definition oracle: supp(i,j) = |S_i ∩ S_j| by sorted merge and by
                 horizontal pair counting; C + OpenMP for speed.
  batmap_ref.py  step-by-step BatMap method in the paper's notation, for
                 byte-level parity of the build and raw-count parity of the intersection.
  fimi.py        NEXT-3: FIMI-repository text -> vertical tidlists (P:56-58, P:556-558,
                 SPEC S:504-512) and the frequent-item pre-filter.
  triples.c      NEXT-4: supp(i,j,k) = |S_i ∩ S_j ∩ S_k| (P:43-44 for itemsets of size 3, the
                 extension P:627-631 leaves open) by three-finger merge and by horizontal
                 triple counting; C + OpenMP.

Parity pins (tests/test_oracle_*.py) tie both to things other than themselves: brute
force on tiny inputs, the Gram matrix X^T X (numpy int64 matmul), the invariant
sum_{i<j} supp = sum_b C(|T_b|, 2), the paper's worked example, the
paper's Fig. 5 indicator assignments, and an exhaustive per-byte check of the SWAR
closed form.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = [os.path.join(_HERE, "pairs.c"), os.path.join(_HERE, "triples.c")]
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/pairs.c + oracle/triples.c -> oracle/liboracle.so (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(s) for s in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11",
                               "-o", tmp, *_SRCS])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        U32 = ctypes.c_uint32
        lib.oracle_merge_count.restype = I64
        lib.oracle_merge_count.argtypes = [P, I64, P, I64]
        lib.oracle_merge_list.restype = None
        lib.oracle_merge_list.argtypes = [P, P, P, P, I64, P]
        lib.oracle_pairs_merge.restype = I64
        lib.oracle_pairs_merge.argtypes = [P, P, P, I64, I64, I64, U32, ctypes.POINTER(P)]
        lib.oracle_pairs_horizontal.restype = I64
        lib.oracle_pairs_horizontal.argtypes = [P, P, I64, I64, P, I64, U32, ctypes.POINTER(P)]
        lib.oracle_free.argtypes = [P]
        lib.oracle_free.restype = None
        lib.oracle_triple_count.restype = I64
        lib.oracle_triple_count.argtypes = [P, I64, P, I64, P, I64]
        lib.oracle_triples_list.restype = None
        lib.oracle_triples_list.argtypes = [P, P, P, P, P, I64, P]
        lib.oracle_triples_horizontal.restype = I64
        lib.oracle_triples_horizontal.argtypes = [P, P, I64, P, I64, U32, ctypes.POINTER(P)]
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _prep(offsets, tids, items):
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    tids = np.ascontiguousarray(tids, dtype=np.int32)
    n = offsets.shape[0] - 1
    if items is None:
        items = np.arange(n, dtype=np.int32)
    else:
        items = np.unique(np.asarray(items, dtype=np.int32))  # ascending, distinct
    return offsets, tids, items


def _take(lib, k: int, outp: ctypes.c_void_p) -> np.ndarray:
    if k < 0:
        raise MemoryError("oracle allocation failed")
    arr = np.ctypeslib.as_array(ctypes.cast(outp, ctypes.POINTER(ctypes.c_uint32)), shape=(max(k, 1) * 3,))
    res = arr[: 3 * k].copy().reshape(k, 3)
    lib.oracle_free(outp)
    return res


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    _load().oracle_set_num_threads(int(n))


def merge_count(a: np.ndarray, b: np.ndarray) -> int:
    """|a ∩ b| for strictly increasing int arrays."""
    lib = _load()
    a = np.ascontiguousarray(a, dtype=np.int32)
    b = np.ascontiguousarray(b, dtype=np.int32)
    return int(lib.oracle_merge_count(_ptr(a), a.shape[0], _ptr(b), b.shape[0]))


def merge_list(offsets, tids, pi, pj) -> np.ndarray:
    """supp for explicit pairs (caller ids) by sorted merge."""
    lib = _load()
    offsets, tids, _ = _prep(offsets, tids, None)
    pi = np.ascontiguousarray(pi, dtype=np.int32)
    pj = np.ascontiguousarray(pj, dtype=np.int32)
    out = np.zeros(pi.shape[0], dtype=np.uint32)
    lib.oracle_merge_list(_ptr(offsets), _ptr(tids), _ptr(pi), _ptr(pj), pi.shape[0], _ptr(out))
    return out


def pairs_merge(offsets, tids, items=None, threshold: int = 1, rows: tuple[int, int] | None = None) -> np.ndarray:
    """Triples (i, j, supp), i<j, supp >= threshold (0 = all), sorted, by sorted merge.

    ``rows`` restricts the first item to selection indices [rows[0], rows[1]) (a sample).
    """
    lib = _load()
    offsets, tids, items = _prep(offsets, tids, items)
    n_sel = items.shape[0]
    rb, re_ = (0, n_sel) if rows is None else rows
    outp = ctypes.c_void_p()
    k = lib.oracle_pairs_merge(_ptr(offsets), _ptr(tids), _ptr(items), n_sel, rb, re_,
                               int(threshold), ctypes.byref(outp))
    return _take(lib, k, outp)


def pairs_horizontal(offsets, tids, m: int, items=None, threshold: int = 1) -> np.ndarray:
    """Triples (i, j, supp), i<j, supp >= threshold (0 = all), sorted, by horizontal counting."""
    lib = _load()
    offsets, tids, items = _prep(offsets, tids, items)
    outp = ctypes.c_void_p()
    k = lib.oracle_pairs_horizontal(_ptr(offsets), _ptr(tids), offsets.shape[0] - 1, int(m),
                                    _ptr(items), items.shape[0], int(threshold), ctypes.byref(outp))
    return _take(lib, k, outp)


# ----------------------------------------------------------------------------- NEXT-4: triples
def triple_count(a: np.ndarray, b: np.ndarray, c: np.ndarray) -> int:
    """|a ∩ b ∩ c| for strictly increasing int arrays (three-finger merge)."""
    lib = _load()
    a, b, c = (np.ascontiguousarray(x, dtype=np.int32) for x in (a, b, c))
    return int(lib.oracle_triple_count(_ptr(a), a.shape[0], _ptr(b), b.shape[0], _ptr(c), c.shape[0]))


def triples_list(offsets, tids, ti, tj, tk) -> np.ndarray:
    """supp(i, j, k) for explicit triples (caller ids) by three-way sorted merge."""
    lib = _load()
    offsets, tids, _ = _prep(offsets, tids, None)
    ti, tj, tk = (np.ascontiguousarray(x, dtype=np.int32) for x in (ti, tj, tk))
    out = np.zeros(ti.shape[0], dtype=np.uint32)
    lib.oracle_triples_list(_ptr(offsets), _ptr(tids), _ptr(ti), _ptr(tj), _ptr(tk), ti.shape[0], _ptr(out))
    return out


def triples_horizontal(offsets, tids, m: int, items=None, threshold: int = 1) -> np.ndarray:
    """Quads (i, j, k, supp), i<j<k, supp >= max(threshold, 1), sorted, by horizontal counting
    (at most 4096 selected items)."""
    lib = _load()
    offsets, tids, items = _prep(offsets, tids, items)
    outp = ctypes.c_void_p()
    k = lib.oracle_triples_horizontal(_ptr(offsets), _ptr(tids), int(m), _ptr(items), items.shape[0],
                                      int(threshold), ctypes.byref(outp))
    if k == -2:
        raise ValueError("triples_horizontal: at most 4096 selected items")
    if k < 0:
        raise MemoryError("oracle allocation failed")
    arr = np.ctypeslib.as_array(ctypes.cast(outp, ctypes.POINTER(ctypes.c_uint32)), shape=(max(k, 1) * 4,))
    res = arr[: 4 * k].copy().reshape(k, 4)
    lib.oracle_free(outp)
    return res
