"""Host-only check of the multi-GPU deal: the planner's per-part
work at N = 2, 4, 8 on the largest configs.

The tile list of the width-class rectangles is cut into parts by batmap_plan_work (no device
needed).  Every part must receive within 1 % of the mean work, counted both as algorithmic
word-compares (sum over the part's pairs of max(W_i, W_j)) and as executed tile compares
(padding included), and the parts together must cover every pair of the triangle exactly once.
The width classes are derived from the seeded instances with the table-range rule of reading
#4 (r_i = max(2^ceil(log2 2|S_i|), 2^s, 128), W = 3r/4)."""
import numpy as np
import pytest

from workloads import make_config


def _classes(name):
    w = make_config(name)
    lens = np.diff(w.offsets)
    s = 0
    while 127 * 2 ** s < w.m:
        s += 1
    r = np.maximum(np.maximum(2 ** np.ceil(np.log2(np.maximum(2 * lens, 1))).astype(np.int64), 2 ** s), 128)
    u, c = np.unique(r, return_counts=True)
    return c.astype(np.int64), (3 * u // 4).astype(np.int64)


@pytest.fixture(scope="module")
def classes():
    return {name: _classes(name) for name in ("C4", "C5_p0.01", "C5_p0.1")}


@pytest.mark.parametrize("name", ["C4", "C5_p0.01", "C5_p0.1"])
@pytest.mark.parametrize("N", [2, 4, 8])
def test_parts_balanced_within_one_percent(classes, name, N):
    from paper_1102_1003_b200 import plan_work

    cn, cw = classes[name]
    _, wc1, _ = plan_work(cn, cw, 0, 1)
    # every pair once: sum over pairs of max(W_i, W_j), computed from the class sizes
    n_tot = np.concatenate([[0], np.cumsum(cn)])
    expect = 0
    for a in range(len(cn)):
        expect += int(cn[a] * (cn[a] - 1) // 2) * int(cw[a])  # within class a
        expect += int(cn[a]) * int(n_tot[a]) * int(cw[a])  # against every narrower item
    assert wc1 == expect
    wcs, tcs = [], []
    for p in range(N):
        _, wc, tc = plan_work(cn, cw, p, N)
        wcs.append(wc)
        tcs.append(tc)
    assert sum(wcs) == wc1  # disjoint parts covering the triangle
    wcs, tcs = np.array(wcs, float), np.array(tcs, float)
    assert wcs.max() / wcs.mean() <= 1.01, wcs
    assert tcs.max() / tcs.mean() <= 1.01, tcs


def test_plan_repeatable_across_threads(classes):
    """The work lists live in a pooled allocator shared by every host thread (plan.cu): plans made
    concurrently from several threads, and again afterwards, are identical."""
    import threading

    from paper_1102_1003_b200 import plan_work

    cn, cw = classes["C4"]
    ref = {N: plan_work(cn, cw, N - 1, N) for N in (1, 3, 8)}
    out, errs = {}, []

    def run(t):
        try:
            for N in (1, 3, 8):
                out[(t, N)] = plan_work(cn, cw, N - 1, N)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=run, args=(t,)) for t in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs
    for (t, N), (items, wc, tc) in out.items():
        assert np.array_equal(items, ref[N][0]) and wc == ref[N][1] and tc == ref[N][2]
