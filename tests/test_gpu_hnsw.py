"""Layered (HNSW) search on the GPU: graphann::search_hnsw
(src/hnsw.cpp:130-147) over layers built by the reference's own build_hnsw,
checked against the reference's search_hnsw. Mirrors acceptance criterion 9
(proj/tests/acceptance.cpp:513-535, a single-layer index searches exactly like
a plain beam search) and uses its desk parameters (m=16, ef=64)."""
import numpy as np
import pytest

from helpers import mixture

pytestmark = pytest.mark.gpu


def _g():
    import paper_2305_04359_b200 as g
    return g


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Oracle, available
    if not available("ref"):
        pytest.skip("the reference build_hnsw/search_hnsw need oracle/_ref")
    return Oracle("ref")


def gpu_layers(data, levels, entry, layers, metric="l2"):
    g = _g()
    idx0 = g.Index(data, metric, layers[0].shape[1])
    idx0.import_graph(layers[0], entry)
    return idx0, g.HnswIndex(idx0, layers[1:], entry)


@pytest.mark.parametrize("dtype,d,metric", [(np.uint8, 32, "l2"), (np.int8, 24, "ip"), (np.float32, 16, "l2")])
@pytest.mark.parametrize("L,k,eps", [(10, 10, 0.0), (64, 10, 0.1), (32, 32, 0.0)])
def test_hnsw_search_parity(ref, dtype, d, metric, L, k, eps):
    """ids, distances, |V| identical to graphann's search_hnsw over the same
    layers (f32: distances within 1e-5 relative, ids equal); REF visited mode
    also reproduces dist_comps summed over all layers."""
    g = _g()
    data, qs = mixture(61, 5000, d, clusters=12, dtype=dtype, nq=300)
    h, levels, entry, layers = ref.hnsw_build(data, 16, 64, metric=metric, workers=4)
    assert len(layers) >= 2, "the test needs upper layers"
    idx0, hn = gpu_layers(data, levels, entry, layers, metric)
    want = ref.hnsw_search(h, data, qs, L, k, eps, metric=metric, workers=4)
    for mode in ("fast", "ref"):
        got = hn.search(qs, g.SearchParams(L, k, eps), visited_mode=mode)
        if dtype == np.float32:
            assert (got.ids == want["ids"]).mean() > 0.999
            np.testing.assert_allclose(got.dists, want["dists"], rtol=1e-5)
        else:
            assert (got.ids == want["ids"]).all()
            assert (got.dists == want["dists"]).all()
            assert (got.n_visited == want["n_visited"]).all()
            if mode == "ref":
                assert (got.dist_comps == want["dist_comps"]).all()
    ref.hnsw_free(h)


def test_single_layer_equals_plain_search(ref):
    """Acceptance criterion 9: with every level forced to 0 the layered search
    is the plain beam search over layer 0 (same ids, dists, |V|, dist_comps)."""
    g = _g()
    data, qs = mixture(62, 4000, 16, clusters=10, dtype=np.float32, nq=200)
    h, levels, entry, layers = ref.hnsw_build(data, 16, 64, single_layer=True, workers=4)
    assert len(layers) == 1 and (levels == 0).all()
    idx0, hn = gpu_layers(data, levels, entry, layers)
    sp = g.SearchParams(64, 10, 0.1)
    a = hn.search(qs, sp, visited_mode="ref")
    b = idx0.search(qs, sp, visited_mode="ref")
    assert (a.ids == b.ids).all() and (a.dists == b.dists).all()
    assert (a.n_visited == b.n_visited).all() and (a.dist_comps == b.dist_comps).all()
    want = ref.hnsw_search(h, data, qs, 64, 10, 0.1, workers=4)
    assert (a.ids == want["ids"]).mean() > 0.999
    ref.hnsw_free(h)


def test_hnsw_validation():
    g = _g()
    data = mixture(63, 200, 8)
    idx0 = g.Index(data, "l2", 8)
    with pytest.raises(ValueError):
        g.HnswIndex(idx0, [np.zeros((100, 4), np.uint32)], 0)      # wrong row count
    with pytest.raises(ValueError):
        g.HnswIndex(idx0, [np.full((200, 4), 500, np.uint32)], 0)  # ids out of range
    with pytest.raises(ValueError):
        g.HnswIndex(idx0, [], 999)                                  # entry out of range
    hn = g.HnswIndex(idx0, [np.full((200, 4), g.GANN_NONE, np.uint32)], 3)
    with pytest.raises(ValueError):
        hn.search(data[:2], g.SearchParams(4, 8, 0.0))              # k > L


def test_run_sweep_over_gpu_indexes(ref, tmp_path):
    """The eval harness over the flat and the layered GPU
    index: every (beam, k, eps) row's recall is graphann's recall_k_at_n of the
    reference's own search results at the same parameters (the ids are equal),
    dist_comps is the per-query mean, and the CSV has graphann's layout."""
    g = _g()
    from paper_2305_04359_b200 import evalutil as E
    data, qs = mixture(64, 5000, 32, clusters=12, nq=200)
    tid, td = ref.groundtruth(data, qs, 20, workers=4)
    adj, start = ref.build(data, 24, 48, 1.2, workers=4)
    idx = g.Index(data, "l2", 24)
    idx.import_graph(adj, start)
    sweep = E.SweepConfig(beams=[10, 32], ks=[10], epsilons=[0.0, 0.1], repetitions=2)
    rep = idx.run_sweep(qs, tid, td, sweep, E.EvalMeta("diskann", "mixture", len(data)))
    assert len(rep.rows) == 4
    for r in rep.rows:
        want = ref.beam_search(adj, start, data, qs, r.beam, r.k, r.epsilon, workers=4)
        assert r.recall == pytest.approx(ref.mean_recall(tid, td, want["ids"], r.k), abs=1e-12)
        got = idx.search(qs, g.SearchParams(r.beam, r.k, r.epsilon))
        assert r.dist_comps == pytest.approx(got.dist_comps.mean())
    assert [(r.recall, r.qps) for r in E.pareto_frontier(rep.rows)] == \
        [(b[3], b[4]) for b in ref.pareto(rep.rows)]
    h, levels, entry, layers = ref.hnsw_build(data, 16, 64, workers=4)
    _, hn = gpu_layers(data, levels, entry, layers)
    hrep = hn.run_sweep(qs, tid, td, sweep, E.EvalMeta("hnsw", "mixture", len(data)))
    for r in hrep.rows:
        want = ref.hnsw_search(h, data, qs, r.beam, r.k, r.epsilon, workers=4)
        assert r.recall == pytest.approx(ref.mean_recall(tid, td, want["ids"], r.k), abs=1e-12)
    ref.hnsw_free(h)
    import io
    buf = io.StringIO()
    E.write_csv(rep, buf)
    ref.write_csv(rep.meta, rep.rows, tmp_path / "r.csv")
    assert buf.getvalue() == (tmp_path / "r.csv").read_text()
