"""NEXT-2 comparison: the sorted-merge path (batmap_merge_pair_supports) per config -- device time,
merge steps/s against the issue-bound ceiling, and exactness against BatMap's result."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1102_1003_b200 import Collection, merge_pair_supports  # noqa: E402
from workloads import make_config  # noqa: E402

for name in sys.argv[1:] or ["C1", "C2"]:
    w = make_config(name)
    o, t = torch.as_tensor(w.offsets).cuda(), torch.as_tensor(w.tids).cuda()
    best = None
    for _ in range(3):
        r, ms, steps = merge_pair_supports(o, t, w.m, threshold=w.threshold, capacity=1 << 20)
        best = ms if best is None or ms < best else best
    c = Collection(o, t, w.m, seed=1)
    bm = c.pair_supports(threshold=w.threshold)
    st = c.stats()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    # issue-bound ceiling: ~10 integer instructions per two-finger step at 128 lanes/clk/SM
    ceiling = 128 / 10 * sms * 1.965e9
    print(json.dumps(dict(config=name, merge_ms=round(best, 3), batmap_pairs_ms=round(st["pairs_ms"], 3),
                          batmap_k2_ms=round(st["k2_ms"], 3), merge_steps=steps,
                          steps_per_s=steps / (best / 1e3), frac_of_issue_ceiling=steps / (best / 1e3) / ceiling,
                          K=int(r.shape[0]), equal_to_batmap=bool(torch.equal(r, bm)))), flush=True)
