#!/usr/bin/env python
"""bench.py -- BatMap all-pairs support counting on B200 (BASELINE.json metric).

One step = one pass of the whole hot path over one synthetic instance resident in HBM:
batmap_build (★K1) + batmap_pair_supports (★K2 intersection + ★K3 corrections/compaction),
plus, for N > 1, the NCCL gather of the compacted triples and their device merge-sort.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl batmap|reference] [--config C2]

N = 1 runs BASELINE configs[1] (C2: uniform, n = 10,000 items, m = 100,000 transactions,
density 1 %, s = 20).  N > 1 (torchrun) scales n by sqrt(N) so that every GPU keeps C2's
number of pair intersections (weak scaling; units = all pairs of the scaled instance).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "item-pair intersections/sec"
UNIT = "pairs/s"


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)), "measured"
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, dev: int):
        self.dev = dev
        self.lines: list[str] = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms", "100", "-i", str(self.dev)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


def _workload(name: str, n_gpus: int, seed: int | None):
    from workloads import make_config

    scale = math.sqrt(n_gpus) if n_gpus > 1 else 1.0
    return make_config(name, scale_items=scale, seed=seed)


def _cpu_baseline(w, target_s: float = 8.0):
    """The oracle (sorted merge, P:59 / P:609-611) as it stands, on a bounded row sample."""
    import oracle

    oracle.set_num_threads(len(os.sched_getaffinity(0)))
    n = w.n
    items = np.arange(n, dtype=np.int32)
    t0 = time.perf_counter()
    probe = 8
    oracle.pairs_merge(w.offsets, w.tids, items, threshold=w.threshold, rows=(0, probe))
    dt = max(time.perf_counter() - t0, 1e-3)
    rows = int(min(n - 1, max(probe, probe * target_s / dt)))
    t0 = time.perf_counter()
    res = oracle.pairs_merge(w.offsets, w.tids, items, threshold=w.threshold, rows=(0, rows))
    dt = time.perf_counter() - t0
    pairs = sum(n - 1 - u for u in range(rows))
    return {"value": pairs / dt, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "cpu_model": _cpu_model(),
            "sample": f"sorted-merge oracle, first {rows} of {n} items x all later items "
                      f"({pairs} pair intersections, {len(res)} frequent) of {w.name}, {dt:.1f} s"}


def _cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle, timed as it stands on this box's host cores."""
    if rank != 0:
        return 0
    import oracle

    oracle.set_num_threads(len(os.sched_getaffinity(0)))  # torchrun exports OMP_NUM_THREADS=1
    w = _workload(args.config, world, args.seed)
    n = w.n
    items = np.arange(n, dtype=np.int32)
    # each step: a bounded row sample (~2-4 s) of the same workload
    t0 = time.perf_counter()
    oracle.pairs_merge(w.offsets, w.tids, items, threshold=w.threshold, rows=(0, 8))
    dt = max(time.perf_counter() - t0, 1e-3)
    rows = int(min(n - 1, max(8, 8 * 3.0 / dt)))
    pairs = sum(n - 1 - u for u in range(rows))
    for _ in range(args.warmup):
        oracle.pairs_merge(w.offsets, w.tids, items, threshold=w.threshold, rows=(0, rows))
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.pairs_merge(w.offsets, w.tids, items, threshold=w.threshold, rows=(0, rows))
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = pairs * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"{w.name}: uniform tidlists, n={n} items (C2 n x sqrt(N)), m={w.m} transactions, "
                               f"p={w.meta.get('p')}, threshold s={w.threshold}", "sample_rows": rows},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": f"sorted-merge oracle, first {rows} of {n} items x all later items "
                                   f"({pairs} pair intersections) per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="batmap", choices=["batmap", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_1102_1003_b200 import Collection, batmap, mine_host
    from paper_1102_1003_b200.dist import build_distributed, gather_triples, mine_distributed

    # test hooks (not used by the driver): run several ranks on one GPU over gloo
    dev_idx = int(os.environ.get("BENCH_FORCE_DEVICE", local_rank))
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    torch.cuda.set_device(dev_idx)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
        else:
            dist.init_process_group(backend)
    n_gpus = world
    w = _workload(args.config, n_gpus, args.seed)
    dev = torch.device("cuda", dev_idx)
    off_d = torch.as_tensor(w.offsets).to(dev)
    tids_d = torch.as_tensor(w.tids).to(dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        if world > 1:  # sharded build + all_gather of the BatMaps
            coll = build_distributed(off_d, tids_d, w.m, seed=1)
        else:
            coll = Collection(off_d, tids_d, w.m, seed=1)
        res = coll.pair_supports(threshold=w.threshold, part=rank, n_parts=world)
        if world > 1:
            allp = gather_triples(res if backend == "nccl" else res.cpu())
            if allp is not None:
                res = batmap.sort_triples(allp.to(dev))
        st = coll.stats()
        coll.close()
        return res, st

    for _ in range(args.warmup):
        res, st = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(dev_idx)
    sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stats = []
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.zero_()  # L2 flush between timed steps, outside the timed events
        ev[k][0].record(stream)
        res, st = step()
        ev[k][1].record(stream)
        stats.append(st)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    n = w.n
    pairs = n * (n - 1) // 2
    value = pairs * args.steps / (tot_ms / 1e3)
    K = int(res.shape[0]) if res is not None else 0

    # ---- dominant kernel roofline: ★K2, plain integer ALU/FMA pipes
    peaks, src = _peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clk_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    peak_cmp = 32.0 * sms * clk_max  # R_int word-compares/s at max clock
    k2_ms = float(np.mean([s["k2_ms"] for s in stats]))
    wc = int(stats[-1]["word_compares"])
    achieved = wc / (k2_ms / 1e3)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "k2_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "alu", "achieved": achieved / 1e12, "peak": peak_cmp / 1e12, "unit": "Tcmp/s",
                "frac": achieved / peak_cmp, "traffic": traffic,
                "kernel": "k2_tiled (BatMap pair intersection)",
                "peak_def": f"R_int = 32 word-compares/clk/SM x {sms} SMs x {clk_max / 1e6:.0f} MHz "
                            f"(sm_max_mhz {src}); 4 integer instructions per 32-bit word compare",
                "k2_share_of_step": float(np.mean([s["k2_ms"] for s in stats])) / (tot_ms / args.steps),
                "k2_ms": k2_ms, "word_compares_per_launch": wc,
                # executed = the kernel's tiles incl. padding (ragged edges, diagonal lower halves);
                # tile_frac is the rate of the inner loop itself, frac the algorithmic one
                "tile_compares_per_launch": int(stats[-1]["tile_compares"]),
                "padding_frac": 1.0 - wc / max(int(stats[-1]["tile_compares"]), 1),
                "tile_frac": int(stats[-1]["tile_compares"]) / (k2_ms / 1e3) / peak_cmp,
                "logical_GBps": 8.0 * wc / (k2_ms / 1e3) / 1e9}

    e2e = None
    cpu = None
    if rank == 0 and world == 1 and not args.no_e2e:
        import torch as _t

        off_h = _t.from_numpy(np.ascontiguousarray(w.offsets)).pin_memory()
        tids_h = _t.from_numpy(np.ascontiguousarray(w.tids)).pin_memory()
        off_np, tids_np = off_h.numpy(), tids_h.numpy()
        cap = K + 1024
        for _ in range(2):
            r = mine_host(off_np, tids_np, w.m, threshold=w.threshold, seed=1, capacity=cap)
        e_ms = []
        for _ in range(max(3, args.steps // 4)):
            flush.zero_()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            r = mine_host(off_np, tids_np, w.m, threshold=w.threshold, seed=1, capacity=cap)
            b.record(stream)
            torch.cuda.synchronize()
            e_ms.append(a.elapsed_time(b))
        assert r.shape[0] == K
        e2e = {"value": pairs / (np.mean(e_ms) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(w.offsets.nbytes + w.tids.nbytes), "d2h_bytes_per_step": int(K * 12),
               "ms_per_step": float(np.mean(e_ms)), "api": "batmap_mine_host (host buffers)"}
    if world > 1 and not args.no_e2e:  # every rank: H2D of the CSR, sharded build, pairs, gather, D2H on rank 0
        import torch as _t

        off_h = _t.from_numpy(np.ascontiguousarray(w.offsets)).pin_memory()
        tids_h = _t.from_numpy(np.ascontiguousarray(w.tids)).pin_memory()
        for _ in range(2):
            r = mine_distributed(off_h, tids_h, w.m, threshold=w.threshold, device=dev, seed=1)
        e_ms = []
        for _ in range(max(3, args.steps // 4)):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            r = mine_distributed(off_h, tids_h, w.m, threshold=w.threshold, device=dev, seed=1)
            b.record(stream)
            torch.cuda.synchronize()
            e_ms.append(a.elapsed_time(b))
        t = torch.tensor([float(np.sum(e_ms))], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_tot = float(t.item())
        if rank == 0:
            assert r.shape[0] == K
            e2e = {"value": pairs * len(e_ms) / (e_tot / 1e3), "unit": UNIT,
                   "h2d_bytes_per_step": int(world * (w.offsets.nbytes + w.tids.nbytes)),
                   "d2h_bytes_per_step": int(K * 12), "ms_per_step": e_tot / len(e_ms),
                   "api": "dist.mine_distributed (host buffers on every rank; max over ranks)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = _cpu_baseline(w)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"{w.name}: uniform tidlists, n={n} items (C2 n x sqrt(N)), m={w.m} "
                                   f"transactions, p={w.meta.get('p')}, threshold s={w.threshold}",
                       "n_items": n, "n_transactions": w.m, "nnz": w.nnz, "threshold": w.threshold,
                       "pairs_per_step": pairs, "frequent_pairs": K, "l2": "flushed (256 MB write) between steps",
                       "parallelism": f"pair-triangle tiles dealt over {world} GPU(s) + NCCL gather"},
            "freq_pairs_per_s": K * args.steps / (tot_ms / 1e3),
            "phases_ms": {"build": float(np.mean([s["build_ms"] for s in stats])),
                          "k1_insert": float(np.mean([s["k1_insert_ms"] for s in stats])),
                          "k1_encode": float(np.mean([s["k1_encode_ms"] for s in stats])),
                          "pairs": float(np.mean([s["pairs_ms"] for s in stats])), "k2": k2_ms,
                          "k3": float(np.mean([s["k3_ms"] for s in stats]))},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(sum(s["launches_build"] + s["launches_pairs"] for s in stats)),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
