"""Build + pair_supports of one config (for profilers): python tools/run_one.py C3 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1102_1003_b200 import Collection
    from workloads import make_config

    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    w = make_config(name)
    o, t = torch.as_tensor(w.offsets).cuda(), torch.as_tensor(w.tids).cuda()
    for _ in range(reps):
        with Collection(o, t, w.m, seed=1) as c:
            k = c.pair_supports(threshold=w.threshold).shape[0]
            s = c.stats()
    print(name, k, {x: round(s[x], 3) for x in ("build_ms", "pairs_ms", "k2_ms", "k3_ms")})


if __name__ == "__main__":
    main()
