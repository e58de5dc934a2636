"""GPU parity of the NEXT-3 row: FIMI text -> vertical tidlists on the device (batmap_fimi_parse),
the frequent-item filter (batmap_fimi_filter / batmap_frequent_items) and mining straight
from a FIMI file, against oracle/fimi.py and the pair oracle.  Bit-exact (integer work)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle.fimi import FimiParseError, filter_csr, frequent_items, parse_fimi  # noqa: E402
from workloads import fimi_text, make_config, uniform, zipf  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _gpu(text, **kw):
    from paper_1102_1003_b200 import parse_fimi as gpu_parse

    db = gpu_parse(text, **kw)
    return (db.offsets.cpu().numpy(), db.tids.cpu().numpy(), db.labels.cpu().numpy().astype(np.uint32), db.m)


def _same(got, ref):
    off, tids, lab, m = got
    ro, rt, rl, rm = ref
    assert m == rm
    np.testing.assert_array_equal(off, ro)
    np.testing.assert_array_equal(tids, rt)
    np.testing.assert_array_equal(lab, rl)


@pytest.mark.parametrize("text", [b"1 2\n2 3\n", b"", b"7 7 9\n", b"\n", b"  ", b"3\r\n4\r\n", b"3\n4", b"\n\n5 5 5\n\n",
                                  b"4294967295 0\n", b"0", b"12 3 12\t\t3 \n 9"])
def test_small_texts(text):
    _same(_gpu(text), parse_fimi(text))


@pytest.mark.parametrize("seed", range(4))
def test_messy_seeded_texts(seed):
    rng = np.random.default_rng(seed)
    off, tids = (uniform(300, 3000, 0.02, seed) if seed % 2 else zipf(2000, 3000, seed=seed))
    labels = np.sort(rng.choice(2 ** 32, size=off.shape[0] - 1, replace=False)).astype(np.int64)
    text = fimi_text(off, tids, 3000, labels=labels, seed=seed, messy=True, final_newline=bool(seed & 2))
    ref = parse_fimi(text)
    _same(_gpu(text), ref)
    # unaligned device text: the same bytes at an odd offset of a larger buffer
    buf = torch.zeros(len(text) + 7, dtype=torch.uint8)
    buf[3:3 + len(text)] = torch.frombuffer(bytearray(text), dtype=torch.uint8)
    _same(_gpu(buf.cuda()[3:3 + len(text)]), ref)


@pytest.mark.parametrize("text", [b"1 2\n3 x\n", b"a", b"1\n2\n\n-4\n", b"1,2\n", b"5\n4294967296\n",
                                  b"1 2 3\n\n\n7 8 9.5", b"1\n" * 5000 + b"2 # 3\n" + b"4\n" * 10])
def test_errors_report_the_oracle_line(text):
    from paper_1102_1003_b200 import BatMapError

    with pytest.raises(FimiParseError) as ref:
        parse_fimi(text)
    with pytest.raises(BatMapError) as got:
        _gpu(text)
    assert f"line {ref.value.line}:" in str(got.value)


@pytest.mark.parametrize("s", [0, 1, 3, 40])
def test_filter_and_frequent_items(s):
    from paper_1102_1003_b200 import frequent_items as gpu_frequent

    off, tids = zipf(3000, 4000, seed=9)
    text = fimi_text(off, tids, 4000, seed=2, messy=True)
    ro, rt, rl, rm = parse_fimi(text)
    keep = frequent_items(ro, s)
    fo, ft = filter_csr(ro, rt, keep)
    _same(_gpu(text, min_support=s), (fo, ft, rl[keep], rm))
    got = gpu_frequent(torch.as_tensor(ro).cuda(), s).cpu().numpy()
    np.testing.assert_array_equal(got, keep)


def test_mine_fimi_end_to_end():
    """Parse + filter + build + pairs from a FIMI file equals the oracle's pairs mapped to labels."""
    from paper_1102_1003_b200 import mine_fimi

    w = make_config("C1")
    labels = np.arange(w.n, dtype=np.int64) * 3 + 1000
    text = fimi_text(w.offsets, w.tids, w.m, labels=labels, seed=5, messy=True)
    got = mine_fimi(text, w.threshold, seed=1)
    np.testing.assert_array_equal(mine_fimi(text, w.threshold / w.m, seed=2), got)  # as a fraction of m
    ro, rt, rl, _ = parse_fimi(text)
    ref = oracle.pairs_horizontal(ro, rt, w.m, threshold=w.threshold).astype(np.int64)
    ref[:, 0] = rl[ref[:, 0]]
    ref[:, 1] = rl[ref[:, 1]]
    np.testing.assert_array_equal(got, ref)


def test_kosarak_shaped_round_trip():
    """At C4's full size (10^6 transactions, 8.1e6 items in ~50 MB of text) the parse is checked by
    the round-trip property pinned in tests/test_oracle_fimi.py: parse(text(CSR)) == CSR restricted
    to the items that occur, labels = ids."""
    w = make_config("C4")
    text = fimi_text(w.offsets, w.tids, w.m, seed=1)
    off, tids, lab, m = _gpu(text)
    keep = np.flatnonzero(np.diff(w.offsets) > 0)
    fo, ft = filter_csr(w.offsets, w.tids, keep)
    assert m == w.m
    np.testing.assert_array_equal(lab, keep.astype(np.uint32))
    np.testing.assert_array_equal(off, fo)
    np.testing.assert_array_equal(tids, ft)


def test_cli_mines_a_fimi_file(tmp_path):
    """batmap_mine <file> <s> (native, C ABI only) prints exactly the oracle's frequent pairs as
    "label_i label_j support" lines."""
    import subprocess

    from paper_1102_1003_b200 import build_ext

    w = make_config("C1")
    labels = np.arange(w.n, dtype=np.int64) * 11 + 3
    path = tmp_path / "c1.dat"
    path.write_bytes(fimi_text(w.offsets, w.tids, w.m, labels=labels, seed=2, messy=True))
    r = subprocess.run([build_ext.build_cli(), str(path), str(w.threshold), "--seed", "3"], capture_output=True,
                       text=True, timeout=120)
    rel = subprocess.run([build_ext.build_cli(), str(path), f"{100.0 * w.threshold / w.m}%", "--quiet"],
                         capture_output=True, text=True, timeout=120)  # the same threshold as a percentage
    assert rel.returncode == 0 and rel.stdout == r.stdout
    assert r.returncode == 0, r.stderr
    got = np.array([list(map(int, ln.split())) for ln in r.stdout.splitlines()], dtype=np.int64).reshape(-1, 3)
    ro, rt, rl, _ = parse_fimi(path.read_bytes())
    ref = oracle.pairs_horizontal(ro, rt, w.m, threshold=w.threshold).astype(np.int64)
    ref[:, 0] = rl[ref[:, 0]]
    ref[:, 1] = rl[ref[:, 1]]
    np.testing.assert_array_equal(got, ref)


def test_select_csr_and_prefiltered_mining():
    """batmap_frequent_items + batmap_select_csr on a Zipf database: the selected CSR equals
    the oracle's restriction, and mining it gives exactly the unfiltered frequent pairs (no pair with
    support >= s contains an infrequent item)."""
    from paper_1102_1003_b200 import Collection, frequent_items as gpu_frequent, select_csr

    off, tids = zipf(4000, 6000, seed=12)
    s = 15
    keep = gpu_frequent(torch.as_tensor(off).cuda(), s)
    ko, kt = select_csr(torch.as_tensor(off).cuda(), torch.as_tensor(tids).cuda(), keep)
    ref_keep = frequent_items(off, s)
    np.testing.assert_array_equal(keep.cpu().numpy(), ref_keep)
    fo, ft = filter_csr(off, tids, ref_keep)
    np.testing.assert_array_equal(ko.cpu().numpy(), fo)
    np.testing.assert_array_equal(kt.cpu().numpy(), ft)
    with Collection(ko, kt, 6000, seed=1) as c:
        got = c.pair_supports(threshold=s).cpu().numpy().astype(np.int64)
    got[:, 0] = ref_keep[got[:, 0]]
    got[:, 1] = ref_keep[got[:, 1]]
    np.testing.assert_array_equal(got, oracle.pairs_horizontal(off, tids, 6000, threshold=s).astype(np.int64))
    empty_o, empty_t = select_csr(torch.as_tensor(off).cuda(), torch.as_tensor(tids).cuda(), np.zeros(0, np.int32))
    assert empty_o.cpu().tolist() == [0] and empty_t.numel() == 0
