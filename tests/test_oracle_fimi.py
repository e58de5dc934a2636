"""Pins of the FIMI reader / frequent-item filter oracle (oracle/fimi.py, NEXT-3 row).

Pinned against things other than the oracle itself: SPEC's worked examples, the
definition S_i = {t : i in T_t} evaluated directly on explicit transaction lists
written out with varied formatting, a round trip through the seeded vertical generators, and a
brute-force count of transactions for the support filter.
"""
import numpy as np
import pytest

from oracle.fimi import FimiParseError, filter_csr, frequent_items, parse_fimi
from workloads import fimi_text, uniform, zipf


def _vertical(transactions):
    """The definition: for each label (ascending) the sorted transaction ids containing it."""
    labels = sorted({x for T in transactions for x in T})
    lists = [[t for t, T in enumerate(transactions) if lab in T] for lab in labels]
    off = np.zeros(len(labels) + 1, np.int64)
    off[1:] = np.cumsum([len(s) for s in lists])
    return off, np.array([t for s in lists for t in s], np.int32), np.array(labels, np.uint32)


def test_spec_examples():
    off, tids, lab, m = parse_fimi(b"1 2\n2 3\n")  # 2 transactions, 3 items
    assert m == 2 and lab.tolist() == [1, 2, 3]
    assert off.tolist() == [0, 1, 3, 4] and tids.tolist() == [0, 0, 1, 1]
    off, tids, lab, m = parse_fimi(b"")  # empty db
    assert m == 0 and lab.size == 0 and off.tolist() == [0] and tids.size == 0
    off, tids, lab, m = parse_fimi(b"7 7 9\n")  # duplicate collapsed -> {7, 9}
    assert m == 1 and lab.tolist() == [7, 9] and tids.tolist() == [0, 0]


@pytest.mark.parametrize("text,m", [(b"\n", 1), (b"1", 1), (b"1\n", 1), (b"1\n\n", 2), (b"  ", 1), (b"\n\n\n", 3),
                                    (b"3\r\n4\r\n", 2), (b"3\n4", 2)])
def test_transaction_count_and_blank_lines(text, m):
    assert parse_fimi(text)[3] == m  # blank lines are empty transactions


def test_definition_on_explicit_transactions():
    rng = np.random.default_rng(0)
    for trial in range(30):
        n_t = int(rng.integers(0, 12))
        T = [set(rng.choice(40, size=int(rng.integers(0, 6)), replace=True).tolist()) for _ in range(n_t)]
        T = [{x * 1_000_003 % 4_000_000_000 for x in s} for s in T]  # large, unordered labels
        seps = [" ", "\t", "  ", " \t"]
        lines = []
        for s in T:
            row = list(s) + (list(s)[:1] if s and rng.random() < 0.5 else [])
            rng.shuffle(row)
            lines.append(seps[trial % 4].join(map(str, row)) + ("\r" if trial % 3 == 0 else ""))
        text = "\n".join(lines) + ("\n" if n_t and trial % 2 else "")
        if n_t and not trial % 2 and lines[-1] == "":
            continue  # an unterminated empty last line is no transaction
        off, tids, lab, m = parse_fimi(text.encode())
        eo, et, el = _vertical(T)
        assert m == n_t
        np.testing.assert_array_equal(lab, el)
        np.testing.assert_array_equal(off, eo)
        np.testing.assert_array_equal(tids, et)


@pytest.mark.parametrize("messy", [False, True])
def test_round_trip_seeded_workloads(messy):
    for off0, tids0, m in [(*uniform(60, 400, 0.05, 3), 400), (*zipf(300, 500, seed=4), 500)]:
        labels = np.arange(off0.shape[0] - 1, dtype=np.int64) * 7 + 5
        text = fimi_text(off0, tids0, m, labels=labels, seed=1, messy=messy, final_newline=not messy)
        off, tids, lab, mm = parse_fimi(text)
        keep = np.flatnonzero(np.diff(off0) > 0)  # items that occur at all
        assert mm == m
        np.testing.assert_array_equal(lab, labels[keep].astype(np.uint32))
        fo, ft = filter_csr(off0, tids0, keep)
        np.testing.assert_array_equal(off, fo)
        np.testing.assert_array_equal(tids, ft)


@pytest.mark.parametrize("text,line", [(b"1 2\n3 x\n", 2), (b"a", 1), (b"1\n2\n\n-4\n", 4), (b"1,2\n", 1),
                                       (b"5\n4294967296\n", 2), (b"1 2 3\n\n\n7 8 9.5", 4)])
def test_errors_carry_the_line(text, line):
    with pytest.raises(FimiParseError) as e:
        parse_fimi(text)
    assert e.value.line == line


def test_largest_label():
    off, tids, lab, m = parse_fimi(b"4294967295 0\n")
    assert lab.tolist() == [0, 4294967295]


def test_frequent_items_brute_force():
    rng = np.random.default_rng(5)
    for _ in range(20):
        T = [set(rng.choice(15, size=int(rng.integers(0, 8)), replace=False).tolist()) for _ in range(25)]
        text = "\n".join(" ".join(map(str, s)) for s in T).encode() + b"\n"
        off, tids, lab, m = parse_fimi(text)
        for s in (0, 1, 3, 7, 26):
            got = frequent_items(off, s)
            expect = [k for k, x in enumerate(lab.tolist()) if sum(x in t for t in T) >= s]
            assert got.tolist() == expect
    assert frequent_items(np.array([0], np.int64), 1).size == 0
