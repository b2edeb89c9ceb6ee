"""The reference's limits, not ours (VERDICT r1 missing #6): the inputs the
reference accepts and round 1 rejected now give graphann's results.

* group_by_key with one key of more than 32,768 pairs (src/semisort.cpp:15-73
  has no size limit): a stable radix sort takes such inputs;
* apply_back_edges on explicit pairs with a hub of 40,000 sources, repeated
  pairs included (src/builder_common.cpp:109-140);
* degree bounds above 256 in the back-edge merge (R = 300 build);
* ground truth with k up to 64 and rows above 256 bytes (src/dataset.cpp:172-217).
"""
import numpy as np
import pytest

from helpers import mixture

pytestmark = pytest.mark.gpu


def _g():
    import paper_2305_04359_b200 as g
    return g


def test_group_by_key_huge_group(oracle):
    g = _g()
    rng = np.random.default_rng(7)
    keys = rng.integers(0, 300, 120_000).astype(np.uint32)
    keys[rng.choice(120_000, 45_000, replace=False)] = 11  # one key of ~45k pairs
    vals = rng.integers(0, 2**32, 120_000, dtype=np.uint64).astype(np.uint32)
    got = g.group_by_key(keys, vals)
    ok, ov, off = oracle.group_by_key(keys, vals)
    ref = {int(ok[off[i]]): ov[off[i]:off[i + 1]].tolist() for i in range(len(off) - 1)}
    mine = {int(got.keys[got.group_offsets[i]]): got.vals[got.group_offsets[i]:got.group_offsets[i + 1]].tolist()
            for i in range(got.groups())}
    assert len(mine[11]) > 32768
    assert mine == ref


def test_apply_back_edges_huge_hub_with_repeats(oracle):
    g = _g()
    data = mixture(14, 60_000, 16, clusters=20)
    adj, start = oracle.build(data[:6000], 16, 32, 1.2, workers=0)
    full = np.full((60_000, 16), 0xFFFFFFFF, np.uint32)
    full[:6000] = adj
    rng = np.random.default_rng(9)
    s = rng.integers(0, 60_000, 50_000).astype(np.uint32)
    t = np.full(50_000, 5, np.uint32)  # one target, 50k sources (some repeated)
    t[:5000] = rng.integers(0, 6000, 5000)
    keep = t != s
    t, s = t[keep], s[keep]
    want = oracle.apply_back_edges(full, data, t, s, 1.2, workers=0)
    idx = g.Index(data, "l2", 16)
    idx.import_graph(full, start)
    idx.apply_back_edges(t, s, g.PruneParams(16, 1.2))
    got, _, _ = idx.export_graph()
    assert (got == want).all(), f"{int((got != want).any(axis=1).sum())} rows differ"


def test_build_degree_bound_above_256(oracle):
    g = _g()
    data = mixture(15, 2500, 16, clusters=6)
    want, ws = oracle.build(data, 300, 320, 1.2, workers=0)
    idx = g.build_diskann(data, "l2", g.DiskannParams(300, 320, 1.2))
    got, _, s = idx.export_graph()
    assert s == ws and (got == want).all(), f"{int((got != want).any(axis=1).sum())} rows differ"


@pytest.mark.parametrize("d,dtype,k", [(128, np.uint8, 50), (320, np.uint8, 10), (400, np.int8, 64),
                                       (600, np.uint8, 32)])
def test_groundtruth_wide_rows_and_large_k(oracle, d, dtype, k):
    g = _g()
    data, qs = mixture(16, 20_000, d, clusters=40, dtype=dtype, nq=200)
    idx = g.Index(data, "l2", 8)
    ids, dists = idx.groundtruth(qs, k)
    wi, wd = oracle.groundtruth(data, qs, k)
    assert (ids == wi).all() and (dists == wd).all()
