"""Small end-to-end case for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every build tier (CTA, cluster of 1/2/4 CTAs over DSMEM, the chunked global tier), serial and
concurrent builds with forced failures, item subsets, a sharded build exchanged in-process, the
cut tail tiles of K2, both K2 tile widths with class promotion, the frequent-item selection, the
GPU merge path, FIMI parsing + filtering + CSR selection, the byte-table K1 tier and the NEXT-4
triples path (candidates, 3-of-4 builds, triple supports), and (not under initcheck, whose reads of
cuBLASLt's output are false positives) the dense path."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from oracle.fimi import filter_csr, parse_fimi as oracle_parse  # noqa: E402
from paper_1102_1003_b200 import (  # noqa: E402
    Collection,
    dense_pair_supports,
    frequent_items,
    merge_pair_supports,
    parse_fimi,
    select_csr,
)
from workloads import fimi_text, uniform, zipf  # noqa: E402

m = 20000
off0, tids0 = uniform(300, m, 0.02, 7)
rng = np.random.default_rng(8)
rows = [tids0[off0[i]:off0[i + 1]] for i in range(len(off0) - 1)]
for size in (3000, 3500, 9000, 17000):  # r = 8192 (cluster of 1), 32768 (2), 65536 (4)
    rows.append(np.sort(rng.choice(m, size=size, replace=False)).astype(np.int32))
off = np.zeros(len(rows) + 1, np.int64)
off[1:] = np.cumsum([len(r) for r in rows])
tids = np.concatenate(rows)
n = len(rows)
ref = oracle.pairs_horizontal(off, tids, m, threshold=2)
o, t = torch.as_tensor(off).cuda(), torch.as_tensor(tids).cuda()
for serial, spread in ((False, "0"), (False, "1"), (True, "1")):
    os.environ["BATMAP_K1_SPREAD"] = spread  # "0": smallest clusters (1/2/4 CTAs); "1": clusters of 8
    c = Collection(o, t, m, seed=3, max_loop=2, serial=serial)  # forced failures exercise K3
    got = c.pair_supports(threshold=2).cpu().numpy().astype(np.uint32)
    assert np.array_equal(got, ref)
    sub = np.arange(0, n, 3, dtype=np.int32)
    got = c.pair_supports(torch.as_tensor(sub).cuda(), threshold=2).cpu().numpy().astype(np.uint32)
    assert np.array_equal(got, oracle.pairs_horizontal(off, tids, m, items=sub, threshold=2))
    c.close()
os.environ.pop("BATMAP_K1_SPREAD")
# sharded build, two parts exchanged in this process
parts = [Collection(o, t, m, seed=4, max_loop=2, part=p, n_parts=2) for p in range(2)]
sw = max(parts[0].shard_sizes(p)[0] for p in range(2))
nf = [c.shard_sizes(c.part)[1] for c in parts]
sf = max(max(nf), 1)
words = torch.zeros(2 * sw, dtype=torch.int32, device="cuda")
fails = torch.zeros(2 * sf, dtype=torch.int64, device="cuda")
for p, c in enumerate(parts):
    c.shard_export(words[p * sw:(p + 1) * sw], fails[p * sf:(p + 1) * sf])
for c in parts:
    c.shard_import(words, sw, fails, nf, sf)
    assert np.array_equal(c.pair_supports(threshold=2).cpu().numpy().astype(np.uint32), ref)
    c.close()
if os.environ.get("SANITIZE_TOOL") != "initcheck":
    d, _ = dense_pair_supports(o, t, m, threshold=2)
    assert np.array_equal(d.cpu().numpy().astype(np.uint32), ref)
# both K2 tile widths (promotion of the small narrow classes included), frequent-only selection
for tn in ("64", "128"):
    os.environ["BATMAP_K2_TN"] = tn
    c = Collection(o, t, m, seed=5, max_loop=2)
    assert np.array_equal(c.pair_supports(threshold=2).cpu().numpy().astype(np.uint32), ref)
    assert np.array_equal(c.pair_supports(threshold=40, frequent_only=True).cpu().numpy().astype(np.uint32),
                          ref[ref[:, 2] >= 40])
    c.close()
os.environ.pop("BATMAP_K2_TN")
# chunked global tier (r = 2^18: 70,000 elements in 35 chunks) next to small items
m2 = 200000
off2, tids2 = uniform(40, m2, 0.005, 9)
rows2 = [tids2[off2[i]:off2[i + 1]] for i in range(len(off2) - 1)]
rows2.append(np.sort(rng.choice(m2, size=70000, replace=False)).astype(np.int32))
off2 = np.zeros(len(rows2) + 1, np.int64)
off2[1:] = np.cumsum([len(r) for r in rows2])
tids2 = np.concatenate(rows2)
c = Collection(torch.as_tensor(off2).cuda(), torch.as_tensor(tids2).cuda(), m2, seed=6, max_loop=1)
assert np.array_equal(c.pair_supports(threshold=1).cpu().numpy().astype(np.uint32),
                      oracle.pairs_horizontal(off2, tids2, m2, threshold=1))
c.close()
# GPU sorted merge
mt, _, _ = merge_pair_supports(o, t, m, threshold=2)
assert np.array_equal(mt.cpu().numpy().astype(np.uint32), ref)
# FIMI ingestion, frequent-item filter, CSR selection
zo, zt = zipf(500, 2000, seed=3)
text = fimi_text(zo, zt, 2000, seed=1, messy=True)
db = parse_fimi(text, min_support=3)
ro, rt, rl, _ = oracle_parse(text)
keep = np.array([i for i in range(len(ro) - 1) if ro[i + 1] - ro[i] >= 3], np.int32)
fo, ft = filter_csr(ro, rt, keep)
assert np.array_equal(db.offsets.cpu().numpy(), fo) and np.array_equal(db.tids.cpu().numpy(), ft)
kd = frequent_items(torch.as_tensor(zo).cuda(), 3)
so, st_ = select_csr(torch.as_tensor(zo).cuda(), torch.as_tensor(zt).cuda(), kd)
eo, et = filter_csr(zo, zt, kd.cpu().numpy())
assert np.array_equal(so.cpu().numpy(), eo) and np.array_equal(st_.cpu().numpy(), et)
# round 2: the byte-table K1 tier on every class (BATMAP_K1_BYTE=all), serial and concurrent
os.environ["BATMAP_K1_BYTE"] = "all"
for serial in (False, True):
    c = Collection(o, t, m, seed=7, max_loop=2, serial=serial)
    assert np.array_equal(c.pair_supports(threshold=2).cpu().numpy().astype(np.uint32), ref)
    c.close()
os.environ.pop("BATMAP_K1_BYTE")
# NEXT-4: Apriori candidates, 3-of-4 BatMaps (concurrent with forced failures, and serial), triple supports
from paper_1102_1003_b200 import Collection3, candidate_triples  # noqa: E402

tri_ref = oracle.triples_horizontal(off, tids, m, threshold=1)
cand = candidate_triples(torch.as_tensor(ref[ref[:, 2] >= 1].astype(np.int32)).cuda(), n)
for serial, ml in ((False, 2), (True, 0)):
    with Collection3(o, t, m, seed=8, max_loop=ml, serial=serial) as c3:
        q = c3.triple_supports(cand, threshold=1).cpu().numpy().astype(np.uint32)
    assert np.array_equal(q, tri_ref), (q.shape, tri_ref.shape)
print("sanitize case ok", len(ref), len(tri_ref))
