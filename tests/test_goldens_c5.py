"""CPU checks of the committed C5 goldens (tests/golden/c5/, written by make_goldens.py from oracle/ only).

The GPU sweep test (test_gpu_c5_sweep.py) trusts these files; here they are checked without
a GPU: integrity (SHA-256 of the stored triples), well-formedness (i < j, sorted by (i, j),
unique, every support >= t_low, the official subset = supp >= s_p as P:43 defines), and, on
the sparse points the oracle recomputes in seconds, reproduction from scratch: the seeded
generator gives the recorded input (CSR hash) and the horizontal oracle gives the stored
triples again, with supp <= min(|S_i|, |S_j|) on every pair.
"""
import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "c5")
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import oracle  # noqa: E402
from make_goldens import T_LOW, csr_sha256, load_triples  # noqa: E402
from workloads import CONFIGS, make_config  # noqa: E402

MANIFEST = json.load(open(os.path.join(GOLD, "manifest.json")))


def test_manifest_has_every_density_point():
    c5 = sorted(k for k in CONFIGS if k.startswith("C5_"))
    assert sorted(MANIFEST) == c5 == sorted(T_LOW)


@pytest.mark.parametrize("name", sorted(MANIFEST))
def test_golden_integrity_and_form(name):
    ent = MANIFEST[name]
    cfg = CONFIGS[name]
    assert ent["key"] == dict(generator=cfg["kind"], n=cfg["n"], m=cfg["m"], p=cfg["p"], seed=cfg["seed"])
    assert ent["threshold"] == cfg["threshold"] and ent["t_low"] == T_LOW[name] <= cfg["threshold"]
    t = load_triples(os.path.join(GOLD, ent["file"]))
    assert t.shape == (ent["K_low"], 3)
    assert hashlib.sha256(np.ascontiguousarray(t, "<u4").tobytes()).hexdigest() == ent["sha256_low"]
    assert np.all(t[:, 0] < t[:, 1]) and np.all(t[:, 1] < cfg["n"])
    key = t[:, 0].astype(np.int64) * cfg["n"] + t[:, 1]
    assert np.all(np.diff(key) > 0)  # sorted by (i, j), no duplicates
    assert np.all(t[:, 2] >= ent["t_low"])
    off = t[t[:, 2] >= ent["threshold"]]
    assert off.shape[0] == ent["K"]
    assert hashlib.sha256(np.ascontiguousarray(off, "<u4").tobytes()).hexdigest() == ent["sha256"]
    # enough pairs to exercise the count distribution near the threshold
    assert ent["K_low"] >= 3e4


@pytest.mark.parametrize("name", ["C5_p0.001", "C5_p0.002"])
def test_golden_reproduces_from_oracle(name):
    ent = MANIFEST[name]
    w = make_config(name)
    assert csr_sha256(w.offsets, w.tids) == ent["csr_sha256"]
    ref = oracle.pairs_horizontal(w.offsets, w.tids, w.m, threshold=ent["t_low"])
    gold = load_triples(os.path.join(GOLD, ent["file"]))
    np.testing.assert_array_equal(ref, gold)
    lens = np.diff(w.offsets)
    assert np.all(gold[:, 2] <= np.minimum(lens[gold[:, 0]], lens[gold[:, 1]]))
