"""Thin Python binding of include/batmap.h (argument marshalling only).

Every step of the hot path runs in libbatmap.so's CUDA kernels; torch provides device
memory and the current stream.  There is no CPU fallback: if the extension is missing
or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbatmap.so")

BATMAP_OK = 0
BATMAP_E_INVALID = -1
BATMAP_E_NOMEM = -2
BATMAP_E_CUDA = -3
BATMAP_E_CAPACITY = -4
BATMAP_E_OVERFLOW = -5
_NAMES = {0: "OK", -1: "E_INVALID", -2: "E_NOMEM", -3: "E_CUDA", -4: "E_CAPACITY", -5: "E_OVERFLOW"}

BATMAP_CHECK_INPUT = 0x1
BATMAP_BUILD_SERIAL = 0x2
BATMAP_PAIRS_RAW = 0x1
BATMAP_PAIRS_SIMPLE = 0x2
BATMAP_PAIRS_FREQUENT = 0x4


class BatMapError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"batmap {_NAMES.get(status, status)}: {msg}")
        self.status = status


class BuildOpts(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("r_min", ctypes.c_uint32), ("max_loop", ctypes.c_uint32),
                ("flags", ctypes.c_uint32), ("reserved", ctypes.c_uint32), ("pi_table", ctypes.c_void_p)]


class Stats(ctypes.Structure):
    _fields_ = [("build_ms", ctypes.c_double), ("k1_insert_ms", ctypes.c_double), ("k1_encode_ms", ctypes.c_double),
                ("pairs_ms", ctypes.c_double), ("k2_ms", ctypes.c_double), ("k3_ms", ctypes.c_double),
                ("word_compares", ctypes.c_int64), ("tile_compares", ctypes.c_int64),
                ("n_candidates", ctypes.c_int64), ("n_results", ctypes.c_int64), ("k2_kind", ctypes.c_int32),
                ("k2_grid", ctypes.c_int32), ("launches_build", ctypes.c_int64), ("launches_pairs", ctypes.c_int64),
                ("build_pre_ms", ctypes.c_double), ("build_post_ms", ctypes.c_double),
                ("k2_tile_cols", ctypes.c_int32), ("reserved", ctypes.c_int32), ("n_selected", ctypes.c_int64)]


class Info(ctypes.Structure):
    _fields_ = [("s_shift", ctypes.c_int32), ("n_classes", ctypes.c_int32), ("U", ctypes.c_int64),
                ("r0", ctypes.c_int64), ("n_items", ctypes.c_int64), ("n_transactions", ctypes.c_int64),
                ("arena_bytes", ctypes.c_int64), ("n_failures", ctypes.c_int64), ("n_failed_tids", ctypes.c_int64)]


class Info3(ctypes.Structure):
    _fields_ = [("s_shift", ctypes.c_int32), ("reserved", ctypes.c_int32), ("r0", ctypes.c_int64),
                ("n_items", ctypes.c_int64), ("n_transactions", ctypes.c_int64), ("arena_bytes", ctypes.c_int64),
                ("n_failures", ctypes.c_int64), ("n_failed_tids", ctypes.c_int64), ("build_ms", ctypes.c_double),
                ("triples_ms", ctypes.c_double)]


_lib = None


def load_library():
    """Load libbatmap.so (built by paper_1102_1003_b200.build_ext); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"CUDA extension not built: {LIB_PATH} is missing "
                           "(run `python -m paper_1102_1003_b200.build_ext`); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
    PI64 = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "batmap_build": ([P, P, I64, I64, ctypes.POINTER(BuildOpts), P, ctypes.POINTER(P)], ctypes.c_int),
        "batmap_build_shard": ([P, P, I64, I64, ctypes.POINTER(BuildOpts), I32, I32, P, ctypes.POINTER(P)],
                               ctypes.c_int),
        "batmap_shard_sizes": ([P, I32, PI64, PI64], ctypes.c_int),
        "batmap_shard_export": ([P, P, I64, P, I64, P], ctypes.c_int),
        "batmap_shard_import": ([P, P, P, P, I64, P, PI64, I64, P], ctypes.c_int),
        "batmap_pair_supports": ([P, P, I64, U32, P, I64, PI64, P], ctypes.c_int),
        "batmap_pair_supports_part": ([P, P, I64, U32, I32, I32, P, I64, PI64, P], ctypes.c_int),
        "batmap_pair_supports_ex": ([P, P, I64, U32, I32, I32, U32, P, I64, PI64, P], ctypes.c_int),
        "batmap_info": ([P, ctypes.POINTER(Info)], ctypes.c_int),
        "batmap_destroy": ([P], None),
        "batmap_last_error": ([], ctypes.c_char_p),
        "batmap_version": ([], ctypes.c_char_p),
        "batmap_mine_host": ([P, P, I64, I64, ctypes.POINTER(BuildOpts), P, I64, U32, P, I64, PI64, P], ctypes.c_int),
        "batmap_export_entries": ([P, I32, P, I64, PI64], ctypes.c_int),
        "batmap_export_failures": ([P, P, P, I64, PI64], ctypes.c_int),
        "batmap_swar_device": ([P, P, I64, P, P], ctypes.c_int),
        "batmap_plan_work": ([I32, P, P, I32, I32, I32, P, I64, PI64, PI64, PI64], ctypes.c_int),
        "batmap_plan_groups": ([I32, P, P, P], ctypes.c_int),
        "batmap_plan_tile": ([I32, P, P, ctypes.POINTER(I32), ctypes.POINTER(I32)], ctypes.c_int),
        "batmap_fimi_parse": ([P, I64, P, ctypes.POINTER(P), PI64], ctypes.c_int),
        "batmap_fimi_info": ([P, PI64, PI64, PI64], ctypes.c_int),
        "batmap_fimi_filter": ([P, U32, P], ctypes.c_int),
        "batmap_fimi_export": ([P, P, P, P, P], ctypes.c_int),
        "batmap_fimi_destroy": ([P], None),
        "batmap_frequent_items": ([P, I64, U32, P, PI64, P], ctypes.c_int),
        "batmap_select_csr": ([P, P, I64, P, I64, P, P, I64, PI64, P], ctypes.c_int),
        "batmap_stats": ([P, ctypes.POINTER(Stats)], ctypes.c_int),
        "batmap_sort_triples": ([P, I64, P], ctypes.c_int),
        "batmap_dense_pair_supports": ([P, P, I64, I64, P, I64, U32, P, I64, PI64, ctypes.POINTER(ctypes.c_double), P],
                                       ctypes.c_int),
        "batmap_merge_pair_supports": ([P, P, I64, I64, P, I64, U32, P, I64, PI64, ctypes.POINTER(ctypes.c_double),
                                        PI64, P], ctypes.c_int),
        "batmap3_build": ([P, P, I64, I64, ctypes.POINTER(BuildOpts), P, ctypes.POINTER(P)], ctypes.c_int),
        "batmap3_triple_supports": ([P, P, I64, U32, P, I64, PI64, P], ctypes.c_int),
        "batmap_candidate_triples": ([P, I64, I64, P, I64, PI64, P], ctypes.c_int),
        "batmap3_info": ([P, ctypes.POINTER(Info3)], ctypes.c_int),
        "batmap3_export_entries": ([P, I32, P, I64, PI64], ctypes.c_int),
        "batmap3_export_failures": ([P, P, P, I64, PI64], ctypes.c_int),
        "batmap3_destroy": ([P], None),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(rc: int, ok=(BATMAP_OK,)):
    if rc not in ok:
        raise BatMapError(rc, load_library().batmap_last_error().decode())
    return rc


def version() -> str:
    return load_library().batmap_version().decode()


def _stream_ptr(stream):
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _dptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _opts(seed, r_min, max_loop, check, pi_table, serial=False):
    o = BuildOpts()
    o.seed = int(seed) & (2 ** 64 - 1)
    o.r_min = int(r_min)
    o.max_loop = int(max_loop)
    o.flags = (BATMAP_CHECK_INPUT if check else 0) | (BATMAP_BUILD_SERIAL if serial else 0)
    o.pi_table = pi_table.data_ptr() if pi_table is not None else None
    return o


class Collection:
    """The BatMaps of one instance on the current CUDA device (batmap_build)."""

    def __init__(self, offsets, tids, n_transactions: int, *, seed: int = 0, r_min: int = 128,
                 max_loop: int = 0, check: bool = False, pi_table=None, serial: bool = False, stream=None,
                 part: int = 0, n_parts: int = 1):
        """part/n_parts > 1: sharded build (batmap_build_shard) -- complete it with shard_export on
        every part, an all_gather, and shard_import (see dist.build_distributed)."""
        import torch

        lib = load_library()
        if not (offsets.is_cuda and tids.is_cuda):
            raise ValueError("offsets and tids must be CUDA tensors")
        self._offsets = offsets.contiguous().to(torch.int64)
        self._tids = tids.contiguous().to(torch.int32)
        self._pi = pi_table.contiguous().to(torch.int32) if pi_table is not None else None
        self.n_items = self._offsets.numel() - 1
        self.m = int(n_transactions)
        self._stream = stream
        opts = _opts(seed, r_min, max_loop, check, self._pi, serial)
        h = ctypes.c_void_p()
        self.part, self.n_parts = int(part), int(n_parts)
        _check(lib.batmap_build_shard(_dptr(self._offsets), _dptr(self._tids), self.n_items, self.m,
                                      ctypes.byref(opts), self.part, self.n_parts, _stream_ptr(stream),
                                      ctypes.byref(h)))
        self._h = h
        self._last_k = 1 << 16
        # the input CSR is not retained by the library (a shard keeps it until shard_import).  The
        # build's last kernels may still read it on the library stream after this call returns:
        # tell the caching allocator, so a converted copy is not reused before they finish.
        if self.n_parts == 1:
            if stream is not None:
                for t in (self._offsets, self._tids):
                    t.record_stream(stream)
            self._offsets = self._tids = None

    # ------------------------------------------------------------------ sharded build
    def shard_sizes(self, part: int):
        """(words of part `part`'s share, failure records of this part or -1)."""
        w, f = ctypes.c_int64(), ctypes.c_int64()
        _check(load_library().batmap_shard_sizes(self._h, int(part), ctypes.byref(w), ctypes.byref(f)))
        return w.value, f.value

    def shard_export(self, words_out, fails_out, stream=None):
        """Write this part's share (int32/uint32 device tensor) and failure records (int64)."""
        _check(load_library().batmap_shard_export(self._h, _dptr(words_out), words_out.numel(), _dptr(fails_out),
                                                  fails_out.numel(), _stream_ptr(stream)))

    def shard_import(self, words_all, stride_words: int, fails_all, n_fails, stride_fails: int, stream=None):
        """Complete the handle from every part's export (blocks of the given strides)."""
        nf = (ctypes.c_int64 * self.n_parts)(*[int(x) for x in n_fails])
        _check(load_library().batmap_shard_import(self._h, _dptr(self._offsets), _dptr(self._tids), _dptr(words_all),
                                                  int(stride_words), _dptr(fails_all), nf, int(stride_fails),
                                                  _stream_ptr(stream)))
        self._offsets = self._tids = None

    def close(self):
        if getattr(self, "_h", None):
            load_library().batmap_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def info(self) -> dict:
        inf = Info()
        _check(load_library().batmap_info(self._h, ctypes.byref(inf)))
        return {k: getattr(inf, k) for k, _ in Info._fields_}

    def stats(self) -> dict:
        """Event-timed phases and work counts of the last build / pair_supports (batmap_stats)."""
        st = Stats()
        _check(load_library().batmap_stats(self._h, ctypes.byref(st)))
        return {k: getattr(st, k) for k, _ in Stats._fields_}

    def pair_supports(self, items=None, threshold: int = 1, *, part: int = 0, n_parts: int = 1,
                      frequent_only: bool = False, raw: bool = False, simple: bool = False, stream=None):
        """int32 tensor [K, 3] of (i, j, support), i < j, support >= threshold, sorted by (i, j).
        frequent_only: intersect only items with |S_i| >= threshold; same output."""
        import torch

        lib = load_library()
        flags = ((BATMAP_PAIRS_RAW if raw else 0) | (BATMAP_PAIRS_SIMPLE if simple else 0) |
                 (BATMAP_PAIRS_FREQUENT if frequent_only else 0))
        it = None
        n_sel = 0
        if items is not None:
            it = items if (hasattr(items, "is_cuda") and items.is_cuda) else torch.as_tensor(np.asarray(items))
            it = it.to(device="cuda", dtype=torch.int32).contiguous()
            n_sel = it.numel()
        st = _stream_ptr(stream if stream is not None else self._stream)
        n_out = ctypes.c_int64(0)
        cap = max(1, self._last_k)
        out = torch.empty((cap, 3), dtype=torch.int32, device="cuda")
        rc = lib.batmap_pair_supports_ex(self._h, _dptr(it), n_sel, int(threshold), part, n_parts, flags,
                                         _dptr(out), cap, ctypes.byref(n_out), st)
        if rc == BATMAP_E_CAPACITY:
            cap = int(n_out.value)
            out = torch.empty((max(cap, 1), 3), dtype=torch.int32, device="cuda")
            rc = lib.batmap_pair_supports_ex(self._h, _dptr(it), n_sel, int(threshold), part, n_parts, flags,
                                             _dptr(out), cap, ctypes.byref(n_out), st)
        _check(rc)
        k = int(n_out.value)
        self._last_k = max(k, 1)
        return out[:k]

    def export_entries(self, item: int) -> np.ndarray:
        """Entry bytes of item's BatMap in entry order (3 r bytes)."""
        lib = load_library()
        r = ctypes.c_int64(0)
        cap = 0
        rc = lib.batmap_export_entries(self._h, int(item), ctypes.c_void_p(1), cap, ctypes.byref(r))
        _check(rc, ok=(BATMAP_OK, BATMAP_E_CAPACITY))
        buf = np.empty(3 * r.value, dtype=np.uint8)
        _check(lib.batmap_export_entries(self._h, int(item), buf.ctypes.data_as(ctypes.c_void_p), buf.size,
                                         ctypes.byref(r)))
        return buf

    def failures(self) -> np.ndarray:
        """F as an int32 array [F, 2] of (item, tid), sorted."""
        lib = load_library()
        n = ctypes.c_int64(0)
        rc = lib.batmap_export_failures(self._h, None, None, 0, ctypes.byref(n))
        _check(rc, ok=(BATMAP_OK, BATMAP_E_CAPACITY))
        items = np.empty(max(n.value, 1), np.int32)
        tids = np.empty(max(n.value, 1), np.int32)
        _check(lib.batmap_export_failures(self._h, items.ctypes.data_as(ctypes.c_void_p),
                                          tids.ctypes.data_as(ctypes.c_void_p), items.size, ctypes.byref(n)))
        return np.stack([items[: n.value], tids[: n.value]], axis=1)


def mine_host(offsets, tids, n_transactions: int, items=None, threshold: int = 1, *, seed: int = 0,
              r_min: int = 128, max_loop: int = 0, capacity: int | None = None, stream=None) -> np.ndarray:
    """End to end on host arrays (batmap_mine_host): returns uint32 [K, 3]."""
    lib = load_library()
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    tids = np.ascontiguousarray(tids, dtype=np.int32)
    it = None if items is None else np.ascontiguousarray(items, dtype=np.int32)
    opts = _opts(seed, r_min, max_loop, False, None)
    cap = int(capacity) if capacity is not None else 1 << 16
    n_out = ctypes.c_int64(0)
    st = _stream_ptr(stream)
    for _ in range(2):
        out = np.empty((max(cap, 1), 3), dtype=np.uint32)
        rc = lib.batmap_mine_host(offsets.ctypes.data_as(ctypes.c_void_p), tids.ctypes.data_as(ctypes.c_void_p),
                                  offsets.shape[0] - 1, int(n_transactions), ctypes.byref(opts),
                                  None if it is None else it.ctypes.data_as(ctypes.c_void_p),
                                  0 if it is None else it.shape[0], int(threshold),
                                  out.ctypes.data_as(ctypes.c_void_p), cap, ctypes.byref(n_out), st)
        if rc != BATMAP_E_CAPACITY:
            break
        cap = int(n_out.value)
    _check(rc)
    return out[: n_out.value]


def dense_pair_supports(offsets, tids, n_transactions: int, items=None, threshold: int = 1, *, stream=None,
                        capacity: int | None = None):
    """NEXT-1 comparison path (batmap_dense_pair_supports): X^T X on the tensor cores.
    Returns (int32 tensor [K, 3] sorted by (i, j), gemm_ms)."""
    import torch

    lib = load_library()
    offsets = offsets.contiguous().to(torch.int64)
    tids = tids.contiguous().to(torch.int32)
    it = None if items is None else torch.as_tensor(np.asarray(items) if not hasattr(items, "is_cuda") else items) \
        .to(device="cuda", dtype=torch.int32).contiguous()
    n_sel = 0 if it is None else it.numel()
    cap = capacity if capacity is not None else 1 << 16
    n_out = ctypes.c_int64(0)
    ms = ctypes.c_double(0)
    for _ in range(2):
        out = torch.empty((max(cap, 1), 3), dtype=torch.int32, device="cuda")
        rc = lib.batmap_dense_pair_supports(_dptr(offsets), _dptr(tids), offsets.numel() - 1, int(n_transactions),
                                            _dptr(it), n_sel, int(threshold), _dptr(out), cap, ctypes.byref(n_out),
                                            ctypes.byref(ms), _stream_ptr(stream))
        if rc != BATMAP_E_CAPACITY:
            break
        cap = int(n_out.value)
    _check(rc)
    return out[: n_out.value], float(ms.value)


def merge_pair_supports(offsets, tids, n_transactions: int, items=None, threshold: int = 1, *, stream=None,
                        capacity: int | None = None):
    """NEXT-2 comparison path (batmap_merge_pair_supports): sorted-list merging.
    Returns (int32 tensor [K, 3] sorted by (i, j), kernel_ms, merge_steps)."""
    import torch

    lib = load_library()
    offsets = offsets.contiguous().to(torch.int64)
    tids = tids.contiguous().to(torch.int32)
    it = None if items is None else torch.as_tensor(np.asarray(items) if not hasattr(items, "is_cuda") else items) \
        .to(device="cuda", dtype=torch.int32).contiguous()
    n_sel = 0 if it is None else it.numel()
    cap = capacity if capacity is not None else 1 << 16
    n_out = ctypes.c_int64(0)
    ms = ctypes.c_double(0)
    steps = ctypes.c_int64(0)
    for _ in range(2):
        out = torch.empty((max(cap, 1), 3), dtype=torch.int32, device="cuda")
        rc = lib.batmap_merge_pair_supports(_dptr(offsets), _dptr(tids), offsets.numel() - 1, int(n_transactions),
                                            _dptr(it), n_sel, int(threshold), _dptr(out), cap, ctypes.byref(n_out),
                                            ctypes.byref(ms), ctypes.byref(steps), _stream_ptr(stream))
        if rc != BATMAP_E_CAPACITY:
            break
        cap = int(n_out.value)
    _check(rc)
    return out[: n_out.value], float(ms.value), int(steps.value)


def sort_triples(t, stream=None):
    """Sort an int32 [K, 3] CUDA tensor of triples in place by (i, j) (batmap_sort_triples)."""
    t = t.contiguous()
    _check(load_library().batmap_sort_triples(_dptr(t), t.shape[0], _stream_ptr(stream)))
    return t


def swar_device(x, y, stream=None):
    """(kernel form, paper form) match counts of word pairs, computed on the device."""
    import torch

    x = x.to(device="cuda", dtype=torch.int32).contiguous()
    y = y.to(device="cuda", dtype=torch.int32).contiguous()
    n = x.numel()
    out = torch.empty(2 * max(n, 1), dtype=torch.int32, device="cuda")
    _check(load_library().batmap_swar_device(_dptr(x), _dptr(y), n, _dptr(out), _stream_ptr(stream)))
    return out[:n], out[n:2 * n]


class FimiDB:
    """A FIMI-repository file parsed on the device (batmap_fimi_parse, optionally filtered by
    batmap_fimi_filter): the vertical CSR ``offsets`` (int64) / ``tids`` (int32) that
    ``Collection`` takes, ``labels`` (int64: dense id -> the file's item label) and ``m``."""

    def __init__(self, offsets, tids, labels, m: int):
        self.offsets, self.tids, self.labels, self.m = offsets, tids, labels, m

    @property
    def n_items(self) -> int:
        return self.offsets.numel() - 1


def parse_fimi(text, min_support: int = 0, *, stream=None) -> FimiDB:
    """FIMI text (bytes, or a uint8 CUDA tensor) -> FimiDB on the device; items with support
    below ``min_support`` dropped.  Raises BatMapError (status E_INVALID, message with
    the line number) on malformed text."""
    import torch

    lib = load_library()
    if isinstance(text, (bytes, bytearray, memoryview)):
        buf = torch.frombuffer(bytearray(text), dtype=torch.uint8) if len(text) else torch.empty(0, dtype=torch.uint8)
        t = buf.pin_memory().to("cuda", non_blocking=True) if len(text) else buf.cuda()
    else:
        t = text.to(device="cuda", dtype=torch.uint8).contiguous()
    h = ctypes.c_void_p()
    bad = ctypes.c_int64(-1)
    _check(lib.batmap_fimi_parse(_dptr(t), t.numel(), _stream_ptr(stream), ctypes.byref(h), ctypes.byref(bad)))
    try:
        if min_support:
            _check(lib.batmap_fimi_filter(h, int(min_support), _stream_ptr(stream)))
        n, nnz, m = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib.batmap_fimi_info(h, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(m)))
        off = torch.empty(n.value + 1, dtype=torch.int64, device="cuda")
        tids = torch.empty(max(nnz.value, 1), dtype=torch.int32, device="cuda")
        lab = torch.empty(max(n.value, 1), dtype=torch.int32, device="cuda")
        _check(lib.batmap_fimi_export(h, _dptr(off), _dptr(tids), _dptr(lab), _stream_ptr(stream)))
        (torch.cuda.current_stream() if stream is None else stream).synchronize()
    finally:
        lib.batmap_fimi_destroy(h)
    labels = lab[: n.value].to(torch.int64) & 0xFFFFFFFF
    return FimiDB(off, tids[: nnz.value], labels, int(m.value))


def frequent_items(offsets, min_support: int, *, stream=None):
    """batmap_frequent_items: int32 CUDA tensor of the ids with |S_i| >= min_support."""
    import torch

    lib = load_library()
    offsets = offsets.to(device="cuda", dtype=torch.int64).contiguous()
    n = offsets.numel() - 1
    out = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    k = ctypes.c_int64(0)
    _check(lib.batmap_frequent_items(_dptr(offsets), n, int(min_support), _dptr(out), ctypes.byref(k),
                                     _stream_ptr(stream)))
    return out[: k.value]


def select_csr(offsets, tids, items, *, stream=None):
    """batmap_select_csr: (offsets int64, tids int32) CUDA tensors of the tidlists of `items`."""
    import torch

    lib = load_library()
    offsets = offsets.to(device="cuda", dtype=torch.int64).contiguous()
    tids = tids.to(device="cuda", dtype=torch.int32).contiguous()
    it = torch.as_tensor(items).to(device="cuda", dtype=torch.int32).contiguous()
    n_sel = it.numel()
    off_out = torch.empty(n_sel + 1, dtype=torch.int64, device="cuda")
    nnz = ctypes.c_int64(0)
    rc = lib.batmap_select_csr(_dptr(offsets), _dptr(tids), offsets.numel() - 1, _dptr(it), n_sel, _dptr(off_out),
                               None, 0, ctypes.byref(nnz), _stream_ptr(stream))
    _check(rc, ok=(BATMAP_OK, BATMAP_E_CAPACITY))
    out = torch.empty(max(nnz.value, 1), dtype=torch.int32, device="cuda")
    _check(lib.batmap_select_csr(_dptr(offsets), _dptr(tids), offsets.numel() - 1, _dptr(it), n_sel, _dptr(off_out),
                                 _dptr(out), out.numel(), ctypes.byref(nnz), _stream_ptr(stream)))
    return off_out, out[: nnz.value]


def mine_fimi(text, threshold, **build_kw) -> np.ndarray:
    """End to end from a FIMI file: parse + frequent-item filter on the device, build the BatMaps
    of the frequent items, emit every pair with support >= threshold.  `threshold` is a count, or
    a float in (0, 1) meaning that fraction of the transactions (ceil).  Returns int64 [K, 3] of
    (label_i, label_j, support), label_i < label_j, sorted."""
    if isinstance(threshold, float) and 0.0 < threshold < 1.0:
        m = parse_fimi(text, min_support=0).m
        threshold = max(1, int(np.ceil(threshold * m - 1e-9)))
    threshold = int(threshold)
    db = parse_fimi(text, min_support=threshold)
    if db.n_items < 2:
        return np.zeros((0, 3), np.int64)
    with Collection(db.offsets, db.tids, max(db.m, 1), **build_kw) as c:
        t = c.pair_supports(threshold=threshold)
    if not t.numel():
        return np.zeros((0, 3), np.int64)
    import torch

    t = t.to(torch.int64)
    return torch.stack([db.labels[t[:, 0]], db.labels[t[:, 1]], t[:, 2]], dim=1).cpu().numpy()


def plan_groups(class_n, class_w):
    """Host-only planner view (batmap_plan_groups): int32 [C] planned class of each input class."""
    lib = load_library()
    cn = np.ascontiguousarray(class_n, dtype=np.int64)
    cw = np.ascontiguousarray(class_w, dtype=np.int64)
    out = np.empty(max(cn.shape[0], 1), dtype=np.int32)
    _check(lib.batmap_plan_groups(cn.shape[0], cn.ctypes.data_as(ctypes.c_void_p), cw.ctypes.data_as(ctypes.c_void_p),
                                  out.ctypes.data_as(ctypes.c_void_p)))
    return out[: cn.shape[0]]


def plan_tile(class_n, class_w):
    """Host-only planner view (batmap_plan_tile): (tile_rows, tile_cols) of the K2 plan."""
    lib = load_library()
    cn = np.ascontiguousarray(class_n, dtype=np.int64)
    cw = np.ascontiguousarray(class_w, dtype=np.int64)
    tr, tc = ctypes.c_int32(), ctypes.c_int32()
    _check(lib.batmap_plan_tile(cn.shape[0], cn.ctypes.data_as(ctypes.c_void_p), cw.ctypes.data_as(ctypes.c_void_p),
                                ctypes.byref(tr), ctypes.byref(tc)))
    return int(tr.value), int(tc.value)


def plan_work(class_n, class_w, part: int = 0, n_parts: int = 1, grid_cap: int = 0):
    """Host-only planner view (batmap_plan_work): (items int32 [T, 8] = (a, b, ti, tj, k0, k1, R, acc),
    word_compares, tile_compares) of `part`."""
    lib = load_library()
    cn = np.ascontiguousarray(class_n, dtype=np.int64)
    cw = np.ascontiguousarray(class_w, dtype=np.int64)
    nt, wc, tcmp = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
    args = (cn.shape[0], cn.ctypes.data_as(ctypes.c_void_p), cw.ctypes.data_as(ctypes.c_void_p), part, n_parts,
            grid_cap)
    rc = lib.batmap_plan_work(*args, None, 0, ctypes.byref(nt), ctypes.byref(wc), ctypes.byref(tcmp))
    _check(rc, ok=(BATMAP_OK, BATMAP_E_CAPACITY))
    items = np.empty((max(nt.value, 1), 8), dtype=np.int32)
    _check(lib.batmap_plan_work(*args, items.ctypes.data_as(ctypes.c_void_p), nt.value, ctypes.byref(nt),
                                ctypes.byref(wc), ctypes.byref(tcmp)))
    return items[: nt.value], int(wc.value), int(tcmp.value)


# ----------------------------------------------------------------------------- NEXT-4: triples
class Collection3:
    """3-of-4 BatMaps of one instance on the current CUDA device (batmap3_build)."""

    def __init__(self, offsets, tids, n_transactions: int, *, seed: int = 0, r_min: int = 128,
                 max_loop: int = 0, check: bool = False, pi_table=None, serial: bool = False, stream=None):
        import torch

        lib = load_library()
        if not (offsets.is_cuda and tids.is_cuda):
            raise ValueError("offsets and tids must be CUDA tensors")
        off = offsets.contiguous().to(torch.int64)
        td = tids.contiguous().to(torch.int32)
        pi = pi_table.contiguous().to(torch.int32) if pi_table is not None else None
        self.n_items = off.numel() - 1
        self._stream = stream
        opts = _opts(seed, r_min, max_loop, check, pi, serial)
        h = ctypes.c_void_p()
        _check(lib.batmap3_build(_dptr(off), _dptr(td), self.n_items, int(n_transactions), ctypes.byref(opts),
                                 _stream_ptr(stream), ctypes.byref(h)))  # synchronises the stream
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            load_library().batmap3_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def info(self) -> dict:
        inf = Info3()
        _check(load_library().batmap3_info(self._h, ctypes.byref(inf)))
        return {k: getattr(inf, k) for k, _ in Info3._fields_}

    def triple_supports(self, triples, threshold: int = 1, stream=None):
        """int32 tensor [K, 4] of (i, j, k, support) for the candidate triples (int32 [n, 3], i < j < k,
        caller ids) with support >= threshold, sorted by (i, j, k)."""
        import torch

        lib = load_library()
        t = triples if (hasattr(triples, "is_cuda") and triples.is_cuda) else torch.as_tensor(np.asarray(triples))
        t = t.to(device="cuda", dtype=torch.int32).contiguous().reshape(-1, 3)
        n = t.shape[0]
        st = _stream_ptr(stream if stream is not None else self._stream)
        n_out = ctypes.c_int64(0)
        cap = max(1, n)
        out = torch.empty((cap, 4), dtype=torch.int32, device="cuda")
        _check(lib.batmap3_triple_supports(self._h, _dptr(t), n, int(threshold), _dptr(out), cap,
                                           ctypes.byref(n_out), st))
        return out[: int(n_out.value)]

    def export_entries(self, item: int) -> np.ndarray:
        lib = load_library()
        r = ctypes.c_int64(0)
        rc = lib.batmap3_export_entries(self._h, int(item), None, 0, ctypes.byref(r))
        _check(rc, ok=(BATMAP_OK, BATMAP_E_CAPACITY))
        buf = np.empty(4 * r.value, dtype=np.uint8)
        _check(lib.batmap3_export_entries(self._h, int(item), buf.ctypes.data_as(ctypes.c_void_p), buf.size,
                                          ctypes.byref(r)))
        return buf

    def failures(self) -> np.ndarray:
        lib = load_library()
        n = ctypes.c_int64(0)
        rc = lib.batmap3_export_failures(self._h, None, None, 0, ctypes.byref(n))
        _check(rc, ok=(BATMAP_OK, BATMAP_E_CAPACITY))
        items = np.empty(max(n.value, 1), np.int32)
        tids = np.empty(max(n.value, 1), np.int32)
        _check(lib.batmap3_export_failures(self._h, items.ctypes.data_as(ctypes.c_void_p),
                                           tids.ctypes.data_as(ctypes.c_void_p), items.size, ctypes.byref(n)))
        return np.stack([items[: n.value], tids[: n.value]], axis=1)


def candidate_triples(pairs, n_items: int, stream=None):
    """Apriori join (batmap_candidate_triples): int32 [C, 3] of i < j < k whose three pairs all occur
    in `pairs` ([K, 3] device int32 triples sorted by (i, j), as Collection.pair_supports returns)."""
    import torch

    lib = load_library()
    p = pairs.to(device="cuda", dtype=torch.int32).contiguous().reshape(-1, 3)
    st = _stream_ptr(stream)
    n_out = ctypes.c_int64(0)
    rc = lib.batmap_candidate_triples(_dptr(p), p.shape[0], int(n_items), None, 0, ctypes.byref(n_out), st)
    _check(rc, ok=(BATMAP_OK, BATMAP_E_CAPACITY))
    cap = int(n_out.value)
    out = torch.empty((max(cap, 1), 3), dtype=torch.int32, device="cuda")
    _check(lib.batmap_candidate_triples(_dptr(p), p.shape[0], int(n_items), _dptr(out), cap, ctypes.byref(n_out), st))
    return out[: int(n_out.value)]


def mine_triples(offsets, tids, n_transactions: int, threshold: int, *, seed: int = 0, stream=None):
    """Frequent triples end to end on the device: frequent pairs (batmap_build + batmap_pair_supports),
    the Apriori candidates (batmap_candidate_triples), 3-of-4 BatMaps (batmap3_build) and their
    supports (batmap3_triple_supports).  Returns (int32 [K3, 4] (i, j, k, support) sorted, dict of
    counts)."""
    with Collection(offsets, tids, n_transactions, seed=seed, stream=stream) as c2:
        pairs = c2.pair_supports(threshold=threshold)
    cand = candidate_triples(pairs, offsets.numel() - 1, stream=stream)
    with Collection3(offsets, tids, n_transactions, seed=seed, stream=stream) as c3:
        quads = c3.triple_supports(cand, threshold=threshold)
        info = c3.info()
    return quads, {"frequent_pairs": int(pairs.shape[0]), "candidates": int(cand.shape[0]),
                   "frequent_triples": int(quads.shape[0]), "build3_ms": info["build_ms"],
                   "triples_ms": info["triples_ms"]}
