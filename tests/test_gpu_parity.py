"""GPU parity: the CUDA path, called through the C-ABI, against the CPU oracle.

The bar is bit-exact equality (integer work): the sorted (i, j, support) triples equal the
definition oracle (sorted merge / horizontal counting, oracle/pairs.c); the BatMap bytes
the build writes equal the step-by-step reference build (oracle/batmap_ref.py); the raw
counts of the intersection kernels equal the reference wrap-around count.
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import batmap_ref as br  # noqa: E402
from workloads import make_config, uniform, zipf  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1102_1003_b200 import batmap

    batmap.load_library()


def _coll(off, tids, m, **kw):
    from paper_1102_1003_b200 import Collection

    return Collection(torch.as_tensor(off, dtype=torch.int64).cuda(), torch.as_tensor(tids, dtype=torch.int32).cuda(),
                      m, **kw)


def _np(t):
    return t.cpu().numpy().astype(np.uint32).reshape(-1, 3)


def _mixed(seed, n=24, m=20000):
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        size = int(min(m - 1, max(1, round(rng.uniform(20, 300) * 2 ** rng.integers(0, 7) / 4))))
        base = np.sort(rng.choice(m, size=size, replace=False))
        if i and rng.random() < 0.5:
            base = np.unique(np.concatenate([base, rows[-1][: size // 2]]))
        rows.append(base.astype(np.int32))
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    return off, np.concatenate(rows), m


# ----------------------------------------------------------------------------- device SWAR
def test_swar_device_exhaustive():
    from paper_1102_1003_b200 import swar_device

    a = np.repeat(np.arange(256, dtype=np.uint64), 256)
    b = np.tile(np.arange(256, dtype=np.uint64), 256)
    rng = np.random.default_rng(1)
    for lane in range(4):
        sh = np.uint64(8 * lane)
        keep = ~(np.uint64(0xFF) << sh) & np.uint64(0xFFFFFFFF)
        x = (rng.integers(0, 2 ** 32, a.shape[0], dtype=np.uint64) & keep) | (a << sh)
        y = (rng.integers(0, 2 ** 32, a.shape[0], dtype=np.uint64) & keep) | (b << sh)
        ref = br.swar_count_np(x, y)
        fast, paper = swar_device(torch.as_tensor(x.astype(np.uint32).view(np.int32)),
                                  torch.as_tensor(y.astype(np.uint32).view(np.int32)))
        np.testing.assert_array_equal(fast.cpu().numpy(), ref)
        np.testing.assert_array_equal(paper.cpu().numpy(), ref)


# ----------------------------------------------------------------------------- K1 bytes
def test_golden_c6_build_and_counts(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "c6_batmap.json")))
    U = g["U"]
    pi = np.array([[(a * x + c) % U for x in range(U)] for a, c in g["pi_affine"]], dtype=np.int32)
    names = ["A", "B", "C"]
    tids = np.concatenate([g["sets"][k] for k in names]).astype(np.int32)
    off = np.zeros(4, np.int64)
    off[1:] = np.cumsum([len(g["sets"][k]) for k in names])
    c = _coll(off, tids, g["m"], r_min=g["r_min"], pi_table=torch.as_tensor(pi).cuda(), serial=True)
    inf = c.info()
    assert inf["s_shift"] == g["s"] and inf["r0"] == g["r0"]
    for i, k in enumerate(names):
        assert " ".join("%02X" % v for v in c.export_entries(i)) == g["bytes"][k]
    assert c.failures().tolist() == [[0, 9]]
    raw = _np(c.pair_supports(threshold=0, raw=True))
    got = {(names[i], names[j]): s for i, j, s in raw.tolist()}
    for pair, val in g["raw_counts"].items():
        if pair[0] != pair[1]:
            assert got[(pair[0], pair[1])] == val
    sup = _np(c.pair_supports(threshold=0))
    assert {(names[i], names[j]): s for i, j, s in sup.tolist()} == {(p[0], p[1]): v for p, v in g["supports"].items()}


@pytest.mark.parametrize("seed,max_loop", [(0, 0), (1, 0), (2, 1), (3, 2)])
def test_build_bytes_equal_reference(seed, max_loop):
    off, tids = uniform(150, 12000, 0.03, 100 + seed)
    c = _coll(off, tids, 12000, seed=seed, max_loop=max_loop, serial=True)
    ref = br.Collection(off, tids, 12000, seed=seed, r_min=128, max_loop=max_loop or None)
    for i in range(ref.n):
        np.testing.assert_array_equal(c.export_entries(i), ref.bytes[i], err_msg=f"item {i}")
    assert c.failures().tolist() == [list(x) for x in ref.failures()]
    if max_loop == 1:
        assert len(ref.failures()) > 0


def test_build_mixed_widths_bytes_and_raw_counts():
    off, tids, m = _mixed(5)
    c = _coll(off, tids, m, seed=9, serial=True)
    ref = br.Collection(off, tids, m, seed=9, r_min=128)
    assert len(set(ref.r)) >= 4
    for i in range(ref.n):
        np.testing.assert_array_equal(c.export_entries(i), ref.bytes[i])
    expect = np.array([(i, j, ref.raw_count(i, j)) for i in range(ref.n) for j in range(i + 1, ref.n)], np.uint32)
    for simple in (False, True):
        np.testing.assert_array_equal(_np(c.pair_supports(threshold=0, raw=True, simple=simple)), expect)


def _check_layout_invariants(c, off, tids, m, seed, r_min=128):
    """Any valid BatMap: every stored element in exactly two tables at its designated
    slots with the right code, exactly one copy flagged (Fig. 5), |S| = stored + failed, and no
    other non-⊥ entry."""
    s, U = br.derive_params(m)
    P = br.pi_table(seed, s)
    fails = {}
    for it, t in c.failures().tolist():
        fails.setdefault(it, set()).add(t)
    r0 = c.info()["r0"]
    for i in range(len(off) - 1):
        S = tids[off[i]:off[i + 1]].tolist()
        ent = c.export_entries(i)
        r = len(ent) // 3
        assert r == br.table_range(len(S), s, r_min)
        seen = np.zeros(len(ent), bool)
        f = fails.get(i, set())
        assert f <= set(S)
        for x in S:
            qs = [br.h(t, int(P[t - 1][x]), r, r0) for t in (1, 2, 3)]
            here = [(t, q) for t, q in zip((1, 2, 3), qs)
                    if ent[q] != br.NULL and (ent[q] & 0x7F) == (int(P[t - 1][x]) >> s)]
            if x in f:
                continue
            assert len(here) == 2, (i, x, here)
            bits = [ent[q] >> 7 for _, q in here]
            (t1, _), (t2, _) = here
            assert bits == [br.indicator(t1, t2), br.indicator(t2, t1)]
            for _, q in here:
                seen[q] = True
        assert int((ent != br.NULL).sum()) == int(seen.sum())  # nothing else stored


@pytest.mark.parametrize("small", ["default", "cluster", "bytes"])
@pytest.mark.parametrize("max_loop", [0, 1])
def test_concurrent_build_invariants(max_loop, small, monkeypatch):
    # small=cluster: no slot-caching CTA tier (uint32 cluster tier down to the smallest tables);
    # small=bytes: every table (r = 256 .. 2^16) in the byte tier
    if small != "default":
        monkeypatch.setenv("BATMAP_K1_SMALL", "cluster")
    if small == "bytes":
        monkeypatch.setenv("BATMAP_K1_BYTE", "all")
    off, tids, m = _mixed(11, n=30)
    c = _coll(off, tids, m, seed=4, max_loop=max_loop)
    _check_layout_invariants(c, off, tids, m, 4)
    if max_loop:
        assert c.info()["n_failures"] > 0
    np.testing.assert_array_equal(_np(c.pair_supports(threshold=0)), oracle.pairs_merge(off, tids, threshold=0))


def _tiers(seed, m=300000, huge=False):
    """Items whose table ranges span the concurrent tiers -- uint32 cluster tier r = 2^14 .. 2^17
    (clusters of 1, 2, 4, 8 CTAs) and global tier r >= 2^18; byte tier r = 2^12 .. 2^19 (clusters of
    1 .. 8 CTAs) and global tier r = 2^20 with `huge` -- plus small items, with shared elements."""
    rng = np.random.default_rng(seed)
    sizes = [5000, 9000, 17000, 40000, 70000, 300, 3000, 8000] + ([150000, 330000] if huge else [])
    base = np.sort(rng.choice(m, size=150000 if huge else 90000, replace=False))
    rows = []
    for k, size in enumerate(sizes):
        own = rng.choice(m, size=size - size // 3, replace=False)
        shared = rng.choice(base, size=size // 3, replace=False)
        rows.append(np.unique(np.concatenate([own, shared])).astype(np.int32))
    off = np.zeros(len(rows) + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    return off, np.concatenate(rows), m


@pytest.mark.parametrize("byte", ["0", "1", "all"])
@pytest.mark.parametrize("spread", ["0", "1"])
@pytest.mark.parametrize("max_loop", [0, 1])
def test_cluster_and_global_tiers(max_loop, spread, byte, monkeypatch):
    # spread=0: the smallest cluster per table size (1, 2, 4, 8 CTAs); spread=1 (default): these
    # one-item classes spread over clusters of 8.  byte=1 (default policy): byte-table tier k1_byte
    # for r = 2^15, 2^16, uint32 cluster tier below, global tier above; byte=all: k1_byte for every
    # class up to r = 2^19 (clusters of up to 8 CTAs); byte=0: the uint32 cluster tier only
    monkeypatch.setenv("BATMAP_K1_SPREAD", spread)
    monkeypatch.setenv("BATMAP_K1_BYTE", byte)
    off, tids, m = _tiers(21, m=600000, huge=byte != "0")
    c = _coll(off, tids, m, seed=6, max_loop=max_loop)
    rs = sorted({len(c.export_entries(i)) // 3 for i in range(len(off) - 1)})
    assert {2 ** 14, 2 ** 15, 2 ** 16, 2 ** 17, 2 ** 18} <= set(rs)
    if byte != "0":
        assert {2 ** 19, 2 ** 20} <= set(rs)
    _check_layout_invariants(c, off, tids, m, 6)
    if max_loop:
        # some item's failure list overflows its 512-entry shared-memory list (kConcFailCap in
        # build.cu), so the global rescan path runs (the total count varies run to run: the
        # concurrent build is nondeterministic, reading #9b)
        per_item = np.bincount(c.failures()[:, 0], minlength=len(off) - 1)
        assert per_item.max() > 512, per_item
    np.testing.assert_array_equal(_np(c.pair_supports(threshold=0)), oracle.pairs_merge(off, tids, threshold=0))


@pytest.mark.parametrize("ipc", ["1", "default"])
@pytest.mark.parametrize("max_loop", [0, 1])
def test_byte_tier_many_small_tables(ipc, max_loop, monkeypatch):
    """A class of 2,500 tiny items in r = 8192 tables (C4's shape): the byte tier builds IPC = 8 items
    per CTA (ipc=default) or one (ipc=1); overlapping sets from a small pool so pairs are frequent."""
    if ipc != "default":
        monkeypatch.setenv("BATMAP_K1_IPC", ipc)
    rng = np.random.default_rng(17)
    m, n = 600000, 2500
    pool = rng.choice(m, size=4000, replace=False)
    rows = []
    for i in range(n):
        size = int(rng.integers(1, 60))
        mine = np.concatenate([rng.choice(pool, size=size // 2, replace=False), rng.choice(m, size=size - size // 2)])
        rows.append(np.unique(mine).astype(np.int32))
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    tids = np.concatenate(rows)
    c = _coll(off, tids, m, seed=9, max_loop=max_loop)
    assert c.info()["n_classes"] == 1 and c.info()["r0"] == 8192
    _check_layout_invariants(c, off, tids, m, 9)
    np.testing.assert_array_equal(_np(c.pair_supports(threshold=2)), oracle.pairs_horizontal(off, tids, m, threshold=2))


@pytest.mark.parametrize("max_loop", [0, 1])
def test_byte_tier_staged_pack(max_loop, monkeypatch):
    """Byte-tier CTAs holding one 96 KB (r = 2^15) or 192 KB (r = 2^16) table each: the staged pack
    (tables written item-major, then k_pack_transpose into the [word][item] arena: one extra launch
    per class) and the direct pack (BATMAP_K1_STAGE=0) both give the oracle's supports and the
    layout invariants, with and without forced failures; 100 + 80 items (one CTA per table on 148
    SMs), so ragged 32-item transpose tiles occur."""
    rng = np.random.default_rng(23)
    m = 200000
    pool = rng.choice(m, size=40000, replace=False)
    rows = []
    for size, cnt in ((12000, 100), (26000, 80)):
        for _ in range(cnt):
            k = int(size * rng.uniform(0.8, 1.0))
            mine = np.concatenate([rng.choice(pool, size=k // 2, replace=False), rng.choice(m, size=k - k // 2)])
            rows.append(np.unique(mine).astype(np.int32))
    off = np.zeros(len(rows) + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    tids = np.concatenate(rows)
    ref = oracle.pairs_horizontal(off, tids, m, threshold=4000)
    launches = {}
    for stage in ("0", "1"):
        monkeypatch.setenv("BATMAP_K1_STAGE", stage)
        c = _coll(off, tids, m, seed=4, max_loop=max_loop)
        assert c.info()["n_classes"] == 2
        launches[stage] = c.stats()["launches_build"]
        _check_layout_invariants(c, off, tids, m, 4)
        np.testing.assert_array_equal(_np(c.pair_supports(threshold=4000)), ref)
        c.close()
    if torch.cuda.get_device_properties(0).multi_processor_count <= 148:  # one CTA per table: both staged
        assert launches["1"] == launches["0"] + 2, launches


def _sharded(off, tids, m, n_parts, **kw):
    """Build every part of a sharded build in this process and exchange as build_distributed
    does (the all_gather is a concatenation here)."""
    from paper_1102_1003_b200 import BatMapError

    parts = [_coll(off, tids, m, part=p, n_parts=n_parts, **kw) for p in range(n_parts)]
    with pytest.raises(BatMapError):
        parts[0].pair_supports(threshold=1)  # incomplete until shard_import
    sw = max(parts[0].shard_sizes(p)[0] for p in range(n_parts))
    assert all(parts[q].shard_sizes(p)[0] == parts[0].shard_sizes(p)[0] for p in range(n_parts) for q in range(n_parts))
    nf = [c.shard_sizes(c.part)[1] for c in parts]
    sf = max(max(nf), 1)
    words = torch.zeros(n_parts * sw, dtype=torch.int32, device="cuda")
    fails = torch.zeros(n_parts * sf, dtype=torch.int64, device="cuda")
    for p, c in enumerate(parts):
        c.shard_export(words[p * sw:(p + 1) * sw], fails[p * sf:(p + 1) * sf])
    for c in parts:
        c.shard_import(words, sw, fails, nf, sf)
    return parts


@pytest.mark.parametrize("n_parts,serial,max_loop", [(2, False, 0), (3, True, 1), (4, False, 1), (5, True, 0)])
def test_sharded_build_exchange(n_parts, serial, max_loop):
    off, tids, m = _mixed(7, n=45)
    parts = _sharded(off, tids, m, n_parts, seed=3, serial=serial, max_loop=max_loop)
    ref = oracle.pairs_merge(off, tids, threshold=1)
    whole = _coll(off, tids, m, seed=3, serial=serial, max_loop=max_loop)
    for c in parts:
        np.testing.assert_array_equal(_np(c.pair_supports(threshold=1)), ref)
        if serial:  # the serial build is deterministic per item: shards reassemble the same bytes
            assert c.info()["n_failures"] == whole.info()["n_failures"]
            for i in range(len(off) - 1):
                np.testing.assert_array_equal(c.export_entries(i), whole.export_entries(i))
    if max_loop:
        assert whole.info()["n_failures"] > 0


def test_sharded_build_tiers_and_parts():
    """Cluster and global tiers split across parts; each rank's share of the pairs after the exchange."""
    off, tids, m = _tiers(5)
    parts = _sharded(off, tids, m, 3, seed=2)
    ref = oracle.pairs_merge(off, tids, threshold=1)
    got = np.concatenate([_np(c.pair_supports(threshold=1, part=c.part, n_parts=3)) for c in parts])
    got = got[np.lexsort((got[:, 1], got[:, 0]))]
    np.testing.assert_array_equal(got, ref)


# ----------------------------------------------------------------------------- end to end
def _check_exact(off, tids, m, thr, items=None, **kw):
    c = _coll(off, tids, m, **kw)
    got = _np(c.pair_supports(items, threshold=thr))
    ref = oracle.pairs_horizontal(off, tids, m, items=items, threshold=thr)
    np.testing.assert_array_equal(got, ref)
    return c, got


def test_c1_exact_both_kernels():
    w = make_config("C1")
    c, got = _check_exact(w.offsets, w.tids, w.m, w.threshold)
    np.testing.assert_array_equal(got, oracle.pairs_merge(w.offsets, w.tids, threshold=w.threshold))
    np.testing.assert_array_equal(_np(c.pair_supports(threshold=w.threshold, simple=True)), got)
    st = c.stats()
    assert st["k2_kind"] == 2  # the last call used the simple kernel
    c.pair_supports(threshold=w.threshold)
    st = c.stats()
    assert st["k2_kind"] == 1 and st["k2_ms"] > 0 and st["word_compares"] > 0


def test_c1_threshold_zero_every_pair():
    w = make_config("C1", scale_items=0.3)
    _check_exact(w.offsets, w.tids, w.m, 0)


@pytest.mark.parametrize("seed", range(6))
def test_mixed_widths_exact_with_failures(seed):
    off, tids, m = _mixed(seed, n=40)
    for max_loop in (0, 1):
        c, _ = _check_exact(off, tids, m, 1, seed=seed, max_loop=max_loop)
        if max_loop == 1:
            assert c.info()["n_failures"] > 0


@pytest.mark.parametrize("ab_cap", ["1", "4096"])
def test_ab_overflow_rerun_exact(ab_cap, monkeypatch):
    """The A_b pass emits into a buffer of a guessed size and re-runs at the exact size when the
    guess is short; BATMAP_AB_CAP forces the guess down so that the re-run path is taken."""
    monkeypatch.setenv("BATMAP_AB_CAP", ab_cap)
    off, tids = uniform(400, 4000, 0.05, 17)
    c, _ = _check_exact(off, tids, 4000, 2, max_loop=1)
    assert c.info()["n_failures"] > 0
    assert len(c.failures()) == c.info()["n_failures"]


def test_colliding_pi_forces_failures_exact():
    off, tids = uniform(60, 3000, 0.1, 5)
    s, U = br.derive_params(3000)
    pi = np.array([[(a * x + cc) % U for x in range(U)] for a, cc in [(1, 0), (5, 3), (11, 7)]], dtype=np.int32)
    c, _ = _check_exact(off, tids, 3000, 1, pi_table=torch.as_tensor(pi).cuda())
    assert c.info()["n_failures"] > 0


def _quest_widths(seed, m=100_000):
    """Width classes shaped like C3's (1, 7, ~40, ~300, ~50, 3 items of r = 2^10 .. 2^15 at
    m = 10^5): small narrow classes that the planner promotes, with shared elements."""
    rng = np.random.default_rng(seed)
    plan = [(1, 300), (7, 700), (40, 1500), (300, 3000), (50, 6000), (3, 12000)]
    pool = np.sort(rng.choice(m, size=20000, replace=False))
    rows = []
    for cnt, size in plan:
        for _ in range(cnt):
            k = int(size * rng.uniform(0.6, 1.0))
            own = rng.choice(m, size=k - k // 4, replace=False)
            shared = rng.choice(pool, size=k // 4, replace=False)
            rows.append(np.unique(np.concatenate([own, shared])).astype(np.int32))
    order = rng.permutation(len(rows))  # ids not in width order
    rows = [rows[k] for k in order]
    off = np.zeros(len(rows) + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    return off, np.concatenate(rows), m


@pytest.mark.parametrize("max_loop", [0, 1])
def test_promoted_classes_exact(max_loop, monkeypatch):
    """Class promotion (small narrow width classes planned as one class of the widest member's
    width, counts divided by K / max(W_i, W_j)): bit-exact against the oracle at thresholds 0, 1
    and 40, on the full selection and on a subset, with and without forced failures; raw counts
    and executed work compared with promotion disabled."""
    off, tids, m = _quest_widths(5)
    c = _coll(off, tids, m, seed=3, max_loop=max_loop)
    if max_loop:
        assert c.info()["n_failures"] > 0
    for thr in (0, 1, 40):
        np.testing.assert_array_equal(_np(c.pair_supports(threshold=thr)), oracle.pairs_merge(off, tids, threshold=thr))
    tc_on = c.stats()["tile_compares"]
    raw_on = _np(c.pair_supports(threshold=0, raw=True))
    sub = np.sort(np.random.default_rng(2).choice(len(off) - 1, size=150, replace=False)).astype(np.int32)
    sub_on = _np(c.pair_supports(items=torch.as_tensor(sub).cuda(), threshold=1))
    np.testing.assert_array_equal(sub_on, oracle.pairs_merge(off, tids, items=sub, threshold=1))
    monkeypatch.setenv("BATMAP_K2_PROMOTE", "0")
    raw_off = _np(c.pair_supports(threshold=0, raw=True))
    tc_off = c.stats()["tile_compares"]
    np.testing.assert_array_equal(raw_on, raw_off)
    assert tc_on < 0.9 * tc_off, (tc_on, tc_off)
    c.close()


@pytest.mark.parametrize("max_loop", [0, 1])
def test_tile_widths_exact(max_loop, monkeypatch):
    """Both K2 tile shapes (128 x 128 pairs per CTA and 128 x 64, BATMAP_K2_TN) on mixed widths with
    and without forced failures: the full selection at thresholds 0 and 3, raw counts, a subset
    and a 3-way part split all equal the oracle / each other."""
    off, tids, m = _quest_widths(8)
    c = _coll(off, tids, m, seed=2, max_loop=max_loop)
    sub = np.sort(np.random.default_rng(4).choice(len(off) - 1, size=200, replace=False)).astype(np.int32)
    ref0 = oracle.pairs_merge(off, tids, threshold=0)
    raws = []
    for tn in ("128", "64"):
        monkeypatch.setenv("BATMAP_K2_TN", tn)
        np.testing.assert_array_equal(_np(c.pair_supports(threshold=0)), ref0)
        assert c.stats()["k2_tile_cols"] == int(tn)
        np.testing.assert_array_equal(_np(c.pair_supports(threshold=3)), ref0[ref0[:, 2] >= 3])
        raws.append(_np(c.pair_supports(threshold=0, raw=True)))
        np.testing.assert_array_equal(_np(c.pair_supports(items=torch.as_tensor(sub).cuda(), threshold=2)),
                                      oracle.pairs_merge(off, tids, items=sub, threshold=2))
        parts = np.concatenate([_np(c.pair_supports(threshold=3, part=p, n_parts=3)) for p in range(3)])
        parts = parts[np.lexsort((parts[:, 1], parts[:, 0]))]
        np.testing.assert_array_equal(parts, ref0[ref0[:, 2] >= 3])
    np.testing.assert_array_equal(raws[0], raws[1])
    c.close()


@pytest.mark.parametrize("tn", ["128", "64"])
def test_balanced_mode_exact(tn, monkeypatch):
    """K2's balanced mode (ragged / diagonal tiles deal their valid blocks' k-steps evenly over the
    warps; ordinary tiles then go through a tail slice) against the default mapping and the oracle,
    on a shape with ragged edges in every class, with and without forced failures, whole and in a
    3-way part split."""
    monkeypatch.setenv("BATMAP_K2_TN", tn)
    off, tids, m = _quest_widths(11)
    ref0 = oracle.pairs_merge(off, tids, threshold=0)
    for max_loop in (0, 1):
        c = _coll(off, tids, m, seed=9, max_loop=max_loop)
        outs = []
        for bal in ("1", "0"):
            monkeypatch.setenv("BATMAP_K2_BALANCE", bal)
            got = _np(c.pair_supports(threshold=0))
            np.testing.assert_array_equal(got, ref0)
            outs.append(_np(c.pair_supports(threshold=0, raw=True)))
            parts = np.concatenate([_np(c.pair_supports(threshold=2, part=p, n_parts=3)) for p in range(3)])
            parts = parts[np.lexsort((parts[:, 1], parts[:, 0]))]
            np.testing.assert_array_equal(parts, ref0[ref0[:, 2] >= 2])
        np.testing.assert_array_equal(outs[0], outs[1])
        c.close()


def test_frequent_only_same_output():
    """BATMAP_PAIRS_FREQUENT intersects only items with |S_i| >= threshold and returns exactly
    the same triples: full selection, a subset, parts, with forced failures; ignored at threshold 0."""
    off, tids = zipf(3000, 5000, seed=21)
    c = _coll(off, tids, 5000, seed=2, max_loop=1)
    sizes = np.diff(off)
    for s in (2, 9, 40):
        ref = oracle.pairs_horizontal(off, tids, 5000, threshold=s)
        np.testing.assert_array_equal(_np(c.pair_supports(threshold=s, frequent_only=True)), ref)
        assert c.stats()["n_selected"] == int((sizes >= s).sum()) < len(sizes)
        parts = np.concatenate([_np(c.pair_supports(threshold=s, frequent_only=True, part=p, n_parts=2))
                                for p in range(2)])
        np.testing.assert_array_equal(parts[np.lexsort((parts[:, 1], parts[:, 0]))], ref)
    sub = np.arange(0, 3000, 3, dtype=np.int32)
    np.testing.assert_array_equal(_np(c.pair_supports(items=torch.as_tensor(sub).cuda(), threshold=5, frequent_only=True)),
                                  oracle.pairs_horizontal(off, tids, 5000, items=sub, threshold=5))
    c.pair_supports(threshold=0, frequent_only=True)
    assert c.stats()["n_selected"] == len(sizes)
    c.close()


def test_items_subset_and_parts():
    w = make_config("C1")
    rng = np.random.default_rng(3)
    items = rng.choice(w.n, size=400, replace=False).astype(np.int32)
    c, got = _check_exact(w.offsets, w.tids, w.m, 3, items=items)
    parts = [_np(c.pair_supports(items, threshold=3, part=p, n_parts=3)) for p in range(3)]
    allp = np.concatenate(parts)
    allp = allp[np.lexsort((allp[:, 1], allp[:, 0]))]
    np.testing.assert_array_equal(allp, got)
    assert sum(len(p) for p in parts) == len(got)


def test_edge_cases():
    from paper_1102_1003_b200 import BatMapError, mine_host

    # empty collection, single item, empty tidlists, threshold above m
    c = _coll(np.zeros(1, np.int64), np.zeros(0, np.int32), 10)
    assert c.pair_supports(threshold=0).shape == (0, 3)
    c = _coll(np.array([0, 3], np.int64), np.array([1, 2, 3], np.int32), 10)
    assert c.pair_supports(threshold=0).shape == (0, 3)
    # items whose tidlists are ALL empty (nnz = 0: the zero-length tids array arrives as NULL)
    off0 = np.zeros(4, np.int64)
    c = _coll(off0, np.zeros(0, np.int32), 10)
    assert c.pair_supports(threshold=0).cpu().numpy().tolist() == [[0, 1, 0], [0, 2, 0], [1, 2, 0]]
    assert c.pair_supports(threshold=1).shape[0] == 0
    from paper_1102_1003_b200 import Collection3, dense_pair_supports, merge_pair_supports

    o0, t0 = torch.as_tensor(off0).cuda(), torch.zeros(0, dtype=torch.int32, device="cuda")
    assert merge_pair_supports(o0, t0, 10, threshold=1)[0].shape[0] == 0
    assert dense_pair_supports(o0, t0, 10, threshold=1)[0].shape[0] == 0
    with Collection3(o0, t0, 10) as c3:
        assert c3.triple_supports(torch.tensor([[0, 1, 2]], dtype=torch.int32), threshold=1).shape[0] == 0
    off = np.array([0, 0, 0, 2], np.int64)
    c, got = _check_exact(off, np.array([0, 5], np.int32), 10, 0)
    assert got.tolist() == [[0, 1, 0], [0, 2, 0], [1, 2, 0]]
    w = make_config("C1", scale_items=0.2)
    _check_exact(w.offsets, w.tids, w.m, w.m + 1)
    # duplicate / out-of-range items are rejected
    c = _coll(w.offsets, w.tids, w.m)
    with pytest.raises(BatMapError):
        c.pair_supports(np.array([1, 1], np.int32))
    with pytest.raises(BatMapError):
        c.pair_supports(np.array([w.n], np.int32))
    # checked mode rejects unsorted / out-of-range tidlists
    with pytest.raises(BatMapError):
        _coll(np.array([0, 2], np.int64), np.array([5, 3], np.int32), 10, check=True)
    with pytest.raises(BatMapError):
        _coll(np.array([0, 1], np.int64), np.array([10], np.int32), 10, check=True)
    # host entry point with the two-call capacity protocol
    res = mine_host(w.offsets, w.tids, w.m, threshold=2, capacity=1)
    np.testing.assert_array_equal(res, oracle.pairs_horizontal(w.offsets, w.tids, w.m, threshold=2))


@pytest.mark.parametrize("m", [1, 2, 126, 127, 128, 254, 255, 1016, 1017])
def test_universe_boundaries(m):
    """Around the code-width boundaries 127 * 2^s (reading #2: s = min{s : 127 * 2^s >= m}; at
    s = 0 every code 0..126 is live and ⊥ = 0x7F must never match): full tidlists (|S| = m),
    identical ones, singletons and random sets, all pairs at threshold 0 and 1, both build modes."""
    rng = np.random.default_rng(m)
    rows = [np.arange(m), np.arange(m), np.array([m - 1]), np.array([0])]
    for _ in range(14):
        k = int(rng.integers(0, m + 1))
        rows.append(np.sort(rng.choice(m, size=k, replace=False)))
    rows.append(rows[-1].copy())
    off = np.zeros(len(rows) + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    tids = np.concatenate(rows).astype(np.int32)
    for serial in (False, True):
        c = _coll(off, tids, m, seed=m, serial=serial)
        for thr in (0, 1):
            np.testing.assert_array_equal(_np(c.pair_supports(threshold=thr)), oracle.pairs_merge(off, tids, threshold=thr))
        c.close()


def test_determinism_and_seed_independence():
    w = make_config("C1")
    a = _coll(w.offsets, w.tids, w.m, seed=1, serial=True)
    b = _coll(w.offsets, w.tids, w.m, seed=1, serial=True)
    for i in range(0, w.n, 97):
        np.testing.assert_array_equal(a.export_entries(i), b.export_entries(i))
    ra = _np(a.pair_supports(threshold=2))
    np.testing.assert_array_equal(ra, _np(b.pair_supports(threshold=2)))
    c = _coll(w.offsets, w.tids, w.m, seed=12345, serial=True)
    assert not np.array_equal(a.export_entries(0), c.export_entries(0))
    np.testing.assert_array_equal(ra, _np(c.pair_supports(threshold=2)))
    d = _coll(w.offsets, w.tids, w.m, seed=1)  # concurrent build: layout may differ, supports may not
    np.testing.assert_array_equal(ra, _np(d.pair_supports(threshold=2)))
    e = _coll(w.offsets, w.tids, w.m, seed=1)  # a second default build: same supports, bytes unspecified
    np.testing.assert_array_equal(ra, _np(e.pair_supports(threshold=2)))


def test_sort_triples():
    from paper_1102_1003_b200 import sort_triples

    rng = np.random.default_rng(0)
    t = rng.integers(0, 1000, size=(5000, 3)).astype(np.int32)
    d = sort_triples(torch.as_tensor(t).cuda())
    ref = t[np.lexsort((t[:, 1], t[:, 0]))]
    np.testing.assert_array_equal(d.cpu().numpy()[:, :2], ref[:, :2])


# ----------------------------------------------------------------------------- full configs
def test_c2_full_exact():
    """The bench workload (BASELINE configs[1]) at full size, in the bench launch configuration."""
    w = make_config("C2")
    c, got = _check_exact(w.offsets, w.tids, w.m, w.threshold)
    assert 1.2e5 < len(got) < 2.5e5
    st = c.stats()
    assert st["k2_kind"] == 1
    # sampled merge cross-check of the horizontal oracle on the emitted pairs
    sel = np.random.default_rng(0).choice(len(got), size=2000, replace=False)
    np.testing.assert_array_equal(oracle.merge_list(w.offsets, w.tids, got[sel, 0], got[sel, 1]), got[sel, 2])


def test_c3_full_exact():
    w = make_config("C3")
    _check_exact(w.offsets, w.tids, w.m, w.threshold)


@pytest.mark.parametrize("name", ["C5_p0.001", "C5_p0.01"])
def test_c5_exact(name):
    w = make_config(name)
    _check_exact(w.offsets, w.tids, w.m, w.threshold)


def test_c4_zipf_exact():
    w = make_config("C4")
    c, got = _check_exact(w.offsets, w.tids, w.m, w.threshold)
    assert c.info()["n_classes"] >= 6


# ----------------------------------------------------------------------------- NEXT-1 dense bitmaps
def _dense(off, tids, m, thr, items=None):
    from paper_1102_1003_b200 import dense_pair_supports

    t, ms = dense_pair_supports(torch.as_tensor(off).cuda(), torch.as_tensor(tids).cuda(), m, items=items, threshold=thr)
    return _np(t), ms


def test_dense_xtx_exact_small_and_subset():
    w = make_config("C1", scale_items=0.3)
    got, _ = _dense(w.offsets, w.tids, w.m, 0)
    np.testing.assert_array_equal(got, oracle.pairs_horizontal(w.offsets, w.tids, w.m, threshold=0))
    w = make_config("C1")
    items = np.random.default_rng(5).choice(w.n, size=333, replace=False).astype(np.int32)
    got, _ = _dense(w.offsets, w.tids, w.m, 2, items=items)
    np.testing.assert_array_equal(got, oracle.pairs_horizontal(w.offsets, w.tids, w.m, items=items, threshold=2))


def test_dense_xtx_c2_equals_batmap():
    w = make_config("C2")
    got, ms = _dense(w.offsets, w.tids, w.m, w.threshold)
    np.testing.assert_array_equal(got, oracle.pairs_horizontal(w.offsets, w.tids, w.m, threshold=w.threshold))
    assert ms > 0


# ----------------------------------------------------------------------------- NEXT-2 sorted merge
def _merge(off, tids, m, thr, items=None):
    from paper_1102_1003_b200 import merge_pair_supports

    t, ms, steps = merge_pair_supports(torch.as_tensor(off).cuda(), torch.as_tensor(tids).cuda(), m, items=items,
                                       threshold=thr)
    return _np(t), ms, steps


def test_merge_exact_small_subset_and_edges():
    w = make_config("C1", scale_items=0.3)
    got, _, steps = _merge(w.offsets, w.tids, w.m, 0)  # every pair, zeros included
    np.testing.assert_array_equal(got, oracle.pairs_horizontal(w.offsets, w.tids, w.m, threshold=0))
    lens = np.diff(w.offsets)
    assert steps == (len(lens) - 1) * int(lens.sum())  # sum over pairs of (a + b)
    w = make_config("C1")
    items = np.random.default_rng(6).choice(w.n, size=600, replace=False).astype(np.int32)
    got, _, _ = _merge(w.offsets, w.tids, w.m, 2, items=items)
    np.testing.assert_array_equal(got, oracle.pairs_horizontal(w.offsets, w.tids, w.m, items=items, threshold=2))
    # empty lists, a single long list against short ones, identical lists, windows refilled many times
    rows = [np.array([], np.int32), np.arange(0, 5000, 1, dtype=np.int32), np.arange(0, 5000, 7, dtype=np.int32),
            np.arange(3, 5000, 7, dtype=np.int32), np.arange(0, 5000, 1, dtype=np.int32), np.array([4999], np.int32)]
    off = np.zeros(len(rows) + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    tids = np.concatenate(rows)
    got, _, _ = _merge(off, tids, 5000, 0)
    np.testing.assert_array_equal(got, oracle.pairs_merge(off, tids, threshold=0))


def test_merge_c2_equals_batmap_and_oracle():
    w = make_config("C2")
    got, ms, _ = _merge(w.offsets, w.tids, w.m, w.threshold)
    np.testing.assert_array_equal(got, oracle.pairs_horizontal(w.offsets, w.tids, w.m, threshold=w.threshold))
    assert ms > 0


@pytest.mark.parametrize("long_len", [9000, 60000])
def test_merge_long_rows_from_global(long_len):
    """Lists too long to stage in shared memory (one S_i + 8 S_j per CTA) take the global-memory
    variant."""
    rng = np.random.default_rng(9)
    m = 200000
    rows = [np.sort(rng.choice(m, size=long_len, replace=False)).astype(np.int32)]
    rows += [np.sort(rng.choice(m, size=int(k), replace=False)).astype(np.int32) for k in rng.integers(10, 3000, 40)]
    off = np.zeros(len(rows) + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    tids = np.concatenate(rows)
    got, _, _ = _merge(off, tids, m, 1)
    np.testing.assert_array_equal(got, oracle.pairs_merge(off, tids, threshold=1))


@pytest.mark.parametrize("case", range(64))
def test_randomized_plans_exact(case, monkeypatch):
    """Randomised stress of the planner features on the device: random item counts, universes,
    size mixes (uniform / Zipf / wide outliers), thresholds, MaxLoop (forced failures), tile width,
    promotion and virtualisation switches, item subsets and part splits -- every result equal to
    the oracle."""
    rng = np.random.default_rng(1000 + case)
    n = int(rng.integers(2, 420))
    m = int(rng.choice([1, 7, 127, 128, 1000, 20000, 60000]))
    kind = case % 3
    rows = []
    for i in range(n):
        if kind == 0:
            k = int(rng.integers(0, min(m, 400) + 1))
        elif kind == 1:
            k = int(min(m, max(0, rng.zipf(1.6) - 1)))
        else:
            k = int(min(m, rng.integers(0, 60) if rng.random() < 0.9 else rng.integers(0, m + 1)))
        rows.append(np.sort(rng.choice(m, size=k, replace=False)).astype(np.int32))
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    tids = np.concatenate(rows) if off[-1] else np.zeros(0, np.int32)
    monkeypatch.setenv("BATMAP_K2_TN", str(rng.choice(["0", "64", "128"])))
    monkeypatch.setenv("BATMAP_K2_PROMOTE", str(rng.choice(["0", "1"])))
    monkeypatch.setenv("BATMAP_K2_VIRTUAL", str(rng.choice(["0", "1"])))
    c = _coll(off, tids, m, seed=int(rng.integers(0, 1 << 30)), max_loop=int(rng.choice([0, 0, 1])))
    thr = int(rng.choice([0, 1, 2, 3, 5]))
    ref = oracle.pairs_merge(off, tids, threshold=thr)
    np.testing.assert_array_equal(_np(c.pair_supports(threshold=thr)), ref)
    if n >= 4:
        sub = np.sort(rng.choice(n, size=int(rng.integers(2, n + 1)), replace=False)).astype(np.int32)
        np.testing.assert_array_equal(_np(c.pair_supports(items=torch.as_tensor(sub).cuda(), threshold=max(thr, 1))),
                                      oracle.pairs_merge(off, tids, items=sub, threshold=max(thr, 1)))
        k = int(rng.integers(2, 5))
        parts = np.concatenate([_np(c.pair_supports(threshold=thr, part=p, n_parts=k)) for p in range(k)])
        parts = parts[np.lexsort((parts[:, 1], parts[:, 0]))] if len(parts) else parts.reshape(0, 3)
        np.testing.assert_array_equal(parts, ref)
    c.close()


def test_c_abi_status_codes_on_device():
    """Status semantics of the C ABI with live device buffers: the two-call capacity protocol of
    pair_supports and select_csr (E_CAPACITY with the required size), out-of-range ids under
    BATMAP_PAIRS_FREQUENT, pair queries on an un-imported shard, NULL outputs of fimi_export."""
    import ctypes

    from paper_1102_1003_b200 import batmap

    lib = batmap.load_library()
    w = make_config("C1")
    o, t = torch.as_tensor(w.offsets).cuda(), torch.as_tensor(w.tids).cuda()
    c = _coll(w.offsets, w.tids, w.m, seed=1)
    ref = oracle.pairs_horizontal(w.offsets, w.tids, w.m, threshold=w.threshold)
    n_out = ctypes.c_int64(-1)
    out = torch.empty((8, 3), dtype=torch.int32, device="cuda")
    st = batmap._stream_ptr(None)
    rc = lib.batmap_pair_supports(c._h, None, 0, w.threshold, batmap._dptr(out), 8, ctypes.byref(n_out), st)
    assert rc == batmap.BATMAP_E_CAPACITY and n_out.value == len(ref)
    big = torch.empty((n_out.value, 3), dtype=torch.int32, device="cuda")
    rc = lib.batmap_pair_supports(c._h, None, 0, w.threshold, batmap._dptr(big), n_out.value, ctypes.byref(n_out), st)
    assert rc == batmap.BATMAP_OK
    np.testing.assert_array_equal(big.cpu().numpy().astype(np.uint32), ref)
    bad = torch.tensor([0, w.n + 5], dtype=torch.int32, device="cuda")
    rc = lib.batmap_pair_supports_ex(c._h, batmap._dptr(bad), 2, 3, 0, 1, batmap.BATMAP_PAIRS_FREQUENT,
                                     batmap._dptr(big), big.shape[0], ctypes.byref(n_out), st)
    assert rc == batmap.BATMAP_E_INVALID and "out of range" in batmap.load_library().batmap_last_error().decode()
    c.close()
    # select_csr two-call protocol
    items = torch.arange(0, w.n, 2, dtype=torch.int32, device="cuda")
    off_out = torch.empty(items.numel() + 1, dtype=torch.int64, device="cuda")
    tids_out = torch.empty(4, dtype=torch.int32, device="cuda")
    nnz = ctypes.c_int64(-1)
    rc = lib.batmap_select_csr(batmap._dptr(o), batmap._dptr(t), w.n, batmap._dptr(items), items.numel(),
                               batmap._dptr(off_out), batmap._dptr(tids_out), 4, ctypes.byref(nnz), st)
    assert rc == batmap.BATMAP_E_CAPACITY
    assert nnz.value == int(np.diff(w.offsets)[::2].sum()) == int(off_out[-1])
    # a shard must be completed (batmap_shard_import) before it is queried
    part = _coll(w.offsets, w.tids, w.m, seed=1, part=0, n_parts=2)
    rc = lib.batmap_pair_supports(part._h, None, 0, 1, batmap._dptr(big), big.shape[0], ctypes.byref(n_out), st)
    assert rc == batmap.BATMAP_E_INVALID
    part.close()
    # fimi_export with NULL outputs copies nothing and succeeds
    text = torch.frombuffer(bytearray(b"1 2\n2 3\n"), dtype=torch.uint8).cuda()
    h, bad_line = ctypes.c_void_p(), ctypes.c_int64()
    assert lib.batmap_fimi_parse(batmap._dptr(text), text.numel(), st, ctypes.byref(h), ctypes.byref(bad_line)) == 0
    assert lib.batmap_fimi_export(h, None, None, None, st) == 0
    lib.batmap_fimi_destroy(h)
