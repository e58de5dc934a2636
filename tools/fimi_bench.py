"""Measure the NEXT-3 row: FIMI text -> vertical CSR on the device (batmap_fimi_parse) and the
frequent-item filter, on text shaped like the paper's FIMI inputs (C4 kosarak-shaped, C3
T40I10D100K-shaped, C2 uniform), against the oracle reader (oracle/fimi.py, pure Python) on a
bounded prefix.  Prints one JSON line per config.

    python tools/fimi_bench.py [C4 C3 C2] [--reps 5]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C4", "C3", "C2"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--oracle-bytes", type=int, default=2_000_000)
    a = ap.parse_args()
    import torch

    from oracle.fimi import parse_fimi as oracle_parse
    from paper_1102_1003_b200 import batmap
    from workloads import fimi_text, make_config

    lib = batmap.load_library()
    st = torch.cuda.current_stream()
    for name in a.configs:
        w = make_config(name)
        text = fimi_text(w.offsets, w.tids, w.m, seed=1)
        dev = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
        host = torch.frombuffer(bytearray(text), dtype=torch.uint8).pin_memory()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        times, times_f, times_e2e = [], [], []
        info = None
        for r in range(a.reps + 2):
            import ctypes

            h, bad = ctypes.c_void_p(), ctypes.c_int64()
            torch.cuda.synchronize()
            e0.record(st)
            batmap._check(lib.batmap_fimi_parse(batmap._dptr(dev), dev.numel(), batmap._stream_ptr(None),
                                                ctypes.byref(h), ctypes.byref(bad)))
            e1.record(st)
            batmap._check(lib.batmap_fimi_filter(h, int(w.threshold), batmap._stream_ptr(None)))
            e2.record(st)
            torch.cuda.synchronize()
            n, nnz, m = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
            batmap._check(lib.batmap_fimi_info(h, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(m)))
            info = (n.value, nnz.value, m.value)
            lib.batmap_fimi_destroy(h)
            # end to end: pinned host text -> device -> parse
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            d2 = host.to("cuda", non_blocking=True)
            batmap._check(lib.batmap_fimi_parse(batmap._dptr(d2), d2.numel(), batmap._stream_ptr(None),
                                                ctypes.byref(h), ctypes.byref(bad)))
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            lib.batmap_fimi_destroy(h)
            del d2
            if r >= 2:
                times.append(e0.elapsed_time(e1))
                times_f.append(e1.elapsed_time(e2))
                times_e2e.append((t1 - t0) * 1e3)
        cut = text.rfind(b"\n", 0, a.oracle_bytes) + 1 or len(text)
        t0 = time.perf_counter()
        oracle_parse(text[:cut])
        t_or = time.perf_counter() - t0
        parse_ms = float(np.median(times))
        print(json.dumps({
            "config": name, "text_MB": len(text) / 1e6, "tokens": int(w.nnz), "transactions": w.m,
            "items_after_parse": int(w.n - (np.diff(w.offsets) == 0).sum()),
            "frequent_items": info[0], "frequent_nnz": info[1], "min_support": int(w.threshold),
            "parse_ms": parse_ms, "parse_GBps": len(text) / parse_ms / 1e6, "filter_ms": float(np.median(times_f)),
            "e2e_host_text_ms": float(np.median(times_e2e)),
            "oracle": {"kind": "oracle/fimi.py (pure Python)", "bytes": cut, "s": t_or,
                       "MBps": cut / t_or / 1e6, "cores": 1},
        }), flush=True)


if __name__ == "__main__":
    main()
