"""CUPTI timeline (torch.profiler) of one batmap3_build (NEXT-4): every kernel, memcpy and memset
with its start offset and duration, and the host runtime calls >= 5 us between them.

    python tools/trace_build3.py [C3]      (BATMAP_K3_SMEM=0: global tier only)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_1102_1003_b200 import Collection3
    from workloads import make_config

    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    w = make_config(name)
    off = torch.as_tensor(w.offsets).cuda()
    tids = torch.as_tensor(w.tids).cuda()
    for _ in range(3):  # warm
        Collection3(off, tids, w.m, seed=1).close()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        c = Collection3(off, tids, w.m, seed=1)
        torch.cuda.synchronize()
    c.close()
    path = f"/tmp/trace3_{name}.json"
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "ts" in e]
    gpu.sort(key=lambda e: e["ts"])
    t0 = gpu[0]["ts"]
    end = t0
    for e in gpu:
        gap = e["ts"] - end
        print(f"{e['ts'] - t0:9.1f} us  +{max(gap, 0):7.1f} gap  {e['dur']:8.1f} us  {e['cat']:10s} {e['name'][:70]}")
        end = max(end, e["ts"] + e["dur"])
    print(f"span {end - t0:.1f} us")
    rt = [e for e in ev if e.get("cat") == "cuda_runtime" and "ts" in e and e["ts"] >= t0 - 50 and e.get("dur", 0) >= 5]
    rt.sort(key=lambda e: e["ts"])
    print("host runtime calls >= 5 us:")
    for e in rt:
        print(f"{e['ts'] - t0:9.1f} us  {e['dur']:8.1f} us  {e['name']}")


if __name__ == "__main__":
    main()
