"""CUPTI timeline (torch.profiler) of one batmap_build + batmap_pair_supports call: every kernel,
memcpy and memset of the library with its start offset and duration, to see where host latency
(syncs, launches) sits between the device work.

    python tools/trace_pairs.py [C1]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_1102_1003_b200 import Collection
    from workloads import make_config

    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    w = make_config(name)
    off = torch.as_tensor(w.offsets).cuda()
    tids = torch.as_tensor(w.tids).cuda()
    for _ in range(3):  # warm
        with Collection(off, tids, w.m, seed=1) as c:
            c.pair_supports(threshold=w.threshold)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        with Collection(off, tids, w.m, seed=1) as c:
            c.pair_supports(threshold=w.threshold)
            st = c.stats()
        torch.cuda.synchronize()
    path = f"/tmp/trace_{name}.json"
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "ts" in e]
    gpu.sort(key=lambda e: e["ts"])
    t0 = gpu[0]["ts"]
    busy = 0.0
    end = t0
    for e in gpu:
        gap = e["ts"] - end
        print(f"{e['ts'] - t0:9.1f} us  +{max(gap, 0):7.1f} gap  {e['dur']:8.1f} us  {e['cat']:10s} {e['name'][:70]}")
        end = max(end, e["ts"] + e["dur"])
        busy += e["dur"]
    print(f"span {end - t0:.1f} us, device busy {busy:.1f} us; stats build {st['build_ms']:.3f} ms pairs {st['pairs_ms']:.3f} ms")
    rt = [e for e in ev if e.get("cat") == "cuda_runtime" and "ts" in e and e["ts"] >= t0 - 50 and e.get("dur", 0) >= 5]
    rt.sort(key=lambda e: e["ts"])
    print("host runtime calls >= 5 us:")
    for e in rt:
        print(f"{e['ts'] - t0:9.1f} us  {e['dur']:8.1f} us  {e['name']}")


if __name__ == "__main__":
    main()
