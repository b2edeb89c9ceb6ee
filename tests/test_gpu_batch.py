"""The several-expansions-per-step search kernel (csrc/search_batch.cuh) against
the CPU oracle. By default it takes beams from L = 320 up; here GANN_BATCH_MIN_L=0
sends every Alg. 1 search {L, L, eps} of the fast visited mode through it, at
small shapes the oracle finishes in seconds: ids, distances, |V| and the visit
sequence must be the reference's (src/search.cpp:62-131), for every step width
and candidate capacity, and a build whose searches run through it must give
the reference's graph bit for bit."""
import os

import numpy as np
import pytest

from helpers import mixture

pytestmark = pytest.mark.gpu


def _g():
    import paper_2305_04359_b200 as g
    return g


@pytest.fixture()
def batch_env():
    keys = ("GANN_BATCH_MIN_L", "GANN_BATCH_EB", "GANN_BATCH_CM", "GANN_BATCH_POLICY", "GANN_GTAB_WIDE")
    old = {k: os.environ.get(k) for k in keys}
    os.environ["GANN_BATCH_MIN_L"] = "0"
    yield os.environ
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _check(got, want, nq):
    assert (got.ids == want["ids"]).all()
    assert (got.dists == want["dists"]).all()
    assert (got.n_visited == want["n_visited"]).all()
    for i in range(nq):
        nv = int(want["n_visited"][i])
        assert (got.visited_ids[i, :nv] == want["visited_ids"][i, :nv]).all()
        assert (got.visited_dists[i, :nv] == want["visited_dists"][i, :nv]).all()


@pytest.mark.parametrize("dtype", [np.uint8, np.int8])
@pytest.mark.parametrize("L", [1, 4, 10, 64, 200, 400])
def test_batch_search_parity_integer(oracle, batch_env, dtype, L):
    g = _g()
    data, qs = mixture(21, 5000, 48, clusters=16, dtype=dtype, nq=300)
    adj, start = oracle.build(data, 24, 48, 1.2, workers=4)
    idx = g.Index(data, "l2", adj.shape[1])
    idx.import_graph(adj, start)
    vcap = 4 * L + 64
    want = oracle.beam_search(adj, start, data, qs, L, L, 0.0, visited_mode=1, vcap=vcap, workers=4)
    stats0 = idx.stats()["merges"]
    got = idx.search(qs, g.SearchParams(L, L, 0.0), visited_mode="fast", vcap=vcap)
    _check(got, want, len(qs))
    assert idx.stats()["merges"] > stats0  # the step counter moved: the batch kernel ran


@pytest.mark.parametrize("eb,cm,policy", [(1, 64, 1), (2, 64, 0), (3, 96, 2), (4, 64, 1), (4, 128, 0), (4, 256, 2)])
def test_batch_step_widths(oracle, batch_env, eb, cm, policy):
    """Every step width / candidate capacity / width policy returns the same search
    (R = 64, the BASELINE degree; eps > 0 with k = L never gates)."""
    g = _g()
    batch_env["GANN_BATCH_EB"] = str(eb)
    batch_env["GANN_BATCH_CM"] = str(cm)
    batch_env["GANN_BATCH_POLICY"] = str(policy)
    data, qs = mixture(22, 6000, 128, clusters=6, nq=200)
    adj, start = oracle.build(data, 64, 96, 1.2, workers=4)
    idx = g.Index(data, "l2", adj.shape[1])
    idx.import_graph(adj, start)
    for L, eps in ((150, 0.0), (330, 0.1)):
        vcap = 4 * L
        want = oracle.beam_search(adj, start, data, qs, L, L, eps, visited_mode=1, vcap=vcap, workers=4)
        got = idx.search(qs, g.SearchParams(L, L, eps), vcap=vcap)
        _check(got, want, len(qs))


def test_batch_default_threshold(oracle):
    """Without any switch the batch kernel takes L >= 320 (and only the Alg. 1 form)."""
    g = _g()
    data, qs = mixture(23, 4000, 64, clusters=8, nq=100)
    adj, start = oracle.build(data, 32, 64, 1.2, workers=4)
    idx = g.Index(data, "l2", adj.shape[1])
    idx.import_graph(adj, start)
    for L, k, batched in ((128, 128, False), (352, 352, True), (352, 10, False)):
        before = idx.stats()["merges"]
        want = oracle.beam_search(adj, start, data, qs, L, k, 0.0, visited_mode=1, workers=4)
        got = idx.search(qs, g.SearchParams(L, k, 0.0))
        assert (got.ids == want["ids"]).all() and (got.n_visited == want["n_visited"]).all()
        assert (idx.stats()["merges"] > before) == batched


def test_batch_search_parity_f32(oracle, batch_env):
    g = _g()
    data, qs = mixture(24, 3000, 200, clusters=10, dtype=np.float32, nq=100)
    adj, start = oracle.build(data, 32, 64, 1.0, metric="ip", workers=4)
    idx = g.Index(data, "ip", adj.shape[1])
    idx.import_graph(adj, start)
    want = oracle.beam_search(adj, start, data, qs, 96, 96, 0.0, metric="ip", workers=4)
    got = idx.search(qs, g.SearchParams(96, 96, 0.0))
    np.testing.assert_allclose(got.dists, want["dists"], rtol=1e-5, atol=1e-5)
    assert (got.ids == want["ids"]).mean() > 0.99


@pytest.mark.parametrize("cap", [0, 400])
def test_batch_build_bit_identical(oracle, batch_env, cap):
    """A build whose searches run through the batch kernel (visit lists in order)
    equals the reference's graph."""
    g = _g()
    data = mixture(25, 6000, 64, clusters=12)
    p = g.DiskannParams(degree_bound=32, build_beam=64, alpha=1.2, max_batch=cap)
    idx = g.build_diskann(data, "l2", p)
    adj, _, start = idx.export_graph()
    ref_adj, ref_start = oracle.build(data, 32, 64, 1.2, cap=cap, workers=4)
    assert start == ref_start
    assert int((adj != ref_adj).any(axis=1).sum()) == 0


@pytest.mark.parametrize("L", [48, 330])
def test_batch_wide_table(oracle, batch_env, L):
    """The visited table's whole-id buckets (taken when n exceeds the u16
    remainders' reach, 2^26 at the default region size; forced here)."""
    g = _g()
    batch_env["GANN_GTAB_WIDE"] = "1"
    data, qs = mixture(26, 5000, 96, clusters=10, nq=200)
    adj, start = oracle.build(data, 48, 64, 1.2, workers=4)
    idx = g.Index(data, "l2", adj.shape[1])
    idx.import_graph(adj, start)
    vcap = 4 * L + 64
    want = oracle.beam_search(adj, start, data, qs, L, L, 0.0, visited_mode=1, vcap=vcap, workers=4)
    got = idx.search(qs, g.SearchParams(L, L, 0.0), vcap=vcap)
    _check(got, want, len(qs))


@pytest.mark.parametrize("n,R", [(2, 1), (9, 3), (40, 8), (300, 33)])
def test_batch_tiny_graphs(oracle, batch_env, n, R):
    """Graphs smaller than the beam (it never fills), rows with one id, an odd degree bound,
    and a vertex without neighbours: the batch kernel's edge cases against the reference."""
    g = _g()
    rng = np.random.default_rng(n)
    data = rng.integers(0, 256, (n, 20)).astype(np.uint8)
    qs = rng.integers(0, 256, (37, 20)).astype(np.uint8)
    adj = np.full((n, R), 0xFFFFFFFF, np.uint32)
    for v in range(n - 1):  # the last vertex keeps an empty row
        nb = rng.permutation([u for u in range(n) if u != v])[: rng.integers(1, R + 1)]
        adj[v, : len(nb)] = nb
    idx = g.Index(data, "l2", R)
    idx.import_graph(adj, 0)
    for L in (1, 5, 64, 400):
        want = oracle.beam_search(adj, 0, data, qs, L, L, 0.0, visited_mode=1, vcap=2 * n + 8, workers=2)
        got = idx.search(qs, g.SearchParams(L, L, 0.0), k_out=min(L, 10), vcap=2 * n + 8)
        kk = min(L, 10)
        assert (got.ids == want["ids"][:, :kk]).all()
        assert (got.n_visited == want["n_visited"]).all()
        for i in range(len(qs)):
            nv = int(want["n_visited"][i])
            assert (got.visited_ids[i, :nv] == want["visited_ids"][i, :nv]).all()
