"""Small end-to-end case for compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1102_1003_b200 import Collection, dense_pair_supports  # noqa: E402
from workloads import uniform  # noqa: E402

off, tids = uniform(300, 20000, 0.02, 7)
m = 20000
ref = oracle.pairs_horizontal(off, tids, m, threshold=2)
o, t = torch.as_tensor(off).cuda(), torch.as_tensor(tids).cuda()
for serial in (False, True):
    c = Collection(o, t, m, seed=3, max_loop=2, serial=serial)  # forced failures exercise K3
    got = c.pair_supports(threshold=2).cpu().numpy().astype(np.uint32)
    assert np.array_equal(got, ref)
    sub = np.arange(0, 300, 3, dtype=np.int32)
    got = c.pair_supports(sub, threshold=2).cpu().numpy().astype(np.uint32)
    assert np.array_equal(got, oracle.pairs_horizontal(off, tids, m, items=sub, threshold=2))
    c.close()
d, _ = dense_pair_supports(o, t, m, threshold=2)
assert np.array_equal(d.cpu().numpy().astype(np.uint32), ref)
print("sanitize case ok", len(ref))
