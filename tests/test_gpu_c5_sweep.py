"""C5 density sweep (BASELINE.json configs[4]) at FULL size, bit-exact on every point.

Every one of the seven density points p in {0.1, 0.2, 0.5, 1, 2, 5, 10} % (n = 20,000 items,
m = 200,000 transactions, P:503-504 generator) runs through the C-ABI in the launch
configuration bench.py uses (default build, default pair kernels) and is compared element
by element with the full-size goldens in tests/golden/c5/.  Those were written by
tests/golden/make_goldens.py, which calls only oracle/ (horizontal pair counting over all
C(20000, 2) pairs, cross-checked by the sorted-merge oracle) -- nothing in them comes from
the CUDA path.

Two thresholds per point: the official s_p of SURVEY §8(d) (inclusive), and a lower
t_low chosen so ~1e5 pairs are emitted and the support distribution just above s_p is
exercised; the official result is the subset supp >= s_p of the t_low golden.
"""
import hashlib
import json
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "c5")
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

from make_goldens import csr_sha256, load_triples  # noqa: E402  (reads goldens; no method arithmetic)
from workloads import make_config  # noqa: E402

MANIFEST = json.load(open(os.path.join(GOLD, "manifest.json")))
POINTS = ["C5_p0.001", "C5_p0.002", "C5_p0.005", "C5_p0.01", "C5_p0.02", "C5_p0.05", "C5_p0.1"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1102_1003_b200 import batmap

    batmap.load_library()


def test_manifest_covers_all_points():
    assert sorted(MANIFEST) == sorted(POINTS)


@pytest.mark.parametrize("name", POINTS)
def test_c5_point_full_size_exact(name):
    from paper_1102_1003_b200 import Collection

    ent = MANIFEST[name]
    w = make_config(name)
    assert w.nnz == ent["nnz"]
    assert csr_sha256(w.offsets, w.tids) == ent["csr_sha256"], "input differs from the golden's input"
    gold_low = load_triples(os.path.join(GOLD, ent["file"]))
    assert gold_low.shape[0] == ent["K_low"]
    assert hashlib.sha256(np.ascontiguousarray(gold_low, "<u4").tobytes()).hexdigest() == ent["sha256_low"]
    gold = gold_low[gold_low[:, 2] >= w.threshold]
    assert gold.shape[0] == ent["K"] and w.threshold == ent["threshold"]

    off_d = torch.as_tensor(w.offsets).cuda()
    tids_d = torch.as_tensor(w.tids).cuda()
    with Collection(off_d, tids_d, w.m) as c:
        del off_d, tids_d  # the handle does not retain the CSR
        for thr, ref in ((w.threshold, gold), (ent["t_low"], gold_low)):
            got = c.pair_supports(threshold=thr).cpu().numpy().astype(np.uint32).reshape(-1, 3)
            assert got.shape == ref.shape, (name, thr, got.shape, ref.shape)
            np.testing.assert_array_equal(got, ref)
