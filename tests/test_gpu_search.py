"""Beam-search parity: CUDA kernel (through the C ABI) vs the CPU oracle.

Mirrors the reference's own search tests (proj/tests/test_search.cpp) and the
SURVEY.md §8c parity protocol: over the reference's own graph the GPU must
return identical neighbor ids, |V| and visit sequences for integer data, and in
REF visited mode the same dist_comps."""
import numpy as np
import pytest

from helpers import mixture

pytestmark = pytest.mark.gpu

SENT = 0xFFFFFFFF


def _g():
    import paper_2305_04359_b200 as g
    return g


def path_fixture(n):
    """1-d points at integer coordinates with path edges i <-> i+1 (test_search.cpp:17-33)."""
    data = np.arange(n, dtype=np.float32).reshape(n, 1)
    adj = np.full((n, 2), SENT, np.uint32)
    for i in range(n):
        nb = ([i - 1] if i > 0 else []) + ([i + 1] if i + 1 < n else [])
        adj[i, : len(nb)] = nb
    return data, adj


def idx_with_graph(data, adj, start, metric="l2"):
    g = _g()
    idx = g.Index(data, metric, adj.shape[1])
    idx.import_graph(adj, start)
    return idx


def test_path_walk_visits_every_hop():  # test_search.cpp:53-62
    g = _g()
    data, adj = path_fixture(5)
    idx = idx_with_graph(data, adj, 0)
    r = idx.search(np.array([[4.2]], np.float32), g.SearchParams(2, 1, 0.0), vcap=8)
    assert r.ids[0, 0] == 4
    assert r.n_visited[0] == 5
    assert list(r.visited_ids[0, :5]) == [0, 1, 2, 3, 4]


def test_k_gate():  # test_search.cpp:64-79
    g = _g()
    data, adj = path_fixture(5)
    idx = idx_with_graph(data, adj, 0)
    q = np.array([[0.1]], np.float32)
    r = idx.search(q, g.SearchParams(4, 1, 0.0), visited_mode="ref", vcap=4)
    assert r.n_visited[0] == 1 and r.visited_ids[0, 0] == 0
    assert r.dist_comps[0] == 2
    r = idx.search(q, g.SearchParams(4, 2, 0.0), vcap=4)
    assert r.n_visited[0] == 2 and r.visited_ids[0, 1] == 1


def test_epsilon_gate():  # test_search.cpp:81-91
    g = _g()
    data, adj = path_fixture(5)
    idx = idx_with_graph(data, adj, 0)
    q = np.array([[0.48]], np.float32)
    assert idx.search(q, g.SearchParams(4, 1, 0.0)).n_visited[0] == 1
    r = idx.search(q, g.SearchParams(4, 1, 0.25), vcap=4)
    assert r.n_visited[0] == 2 and r.visited_ids[0, 1] == 1 and r.ids[0, 0] == 0


def test_saturation_complete_graph_is_exact(oracle):  # test_search.cpp:93-110
    g = _g()
    rng = np.random.default_rng(101)
    n = 300
    data = rng.uniform(0, 1, (n, 4)).astype(np.float32)
    adj = np.array([[u for u in range(n) if u != v] for v in range(n)], np.uint32)
    idx = idx_with_graph(data, adj, 0)
    qs = rng.uniform(0, 1, (50, 4)).astype(np.float32)
    r = idx.search(qs, g.SearchParams(300, 10, 0.0))
    gt_ids, _ = oracle.groundtruth(data, qs, 10)
    assert (r.ids == gt_ids).all()


def test_saturation_ring_is_exact(oracle):  # test_search.cpp:111-126
    g = _g()
    n = 500
    data = np.arange(n, dtype=np.float32).reshape(n, 1)
    adj = np.array([[(i + n - 1) % n, (i + 1) % n] for i in range(n)], np.uint32)
    idx = idx_with_graph(data, adj, 0)
    rng = np.random.default_rng(3)
    qs = rng.uniform(0, n - 1, (20, 1)).astype(np.float32)
    r = idx.search(qs, g.SearchParams(n, 10, 0.0))
    gt_ids, _ = oracle.groundtruth(data, qs, 10)
    assert (r.ids == gt_ids).all()


def test_ties_rank_by_smaller_id():  # test_search.cpp:154-165
    g = _g()
    data = np.array([[0.0], [1.0], [1.0], [2.0]], np.float32)
    adj = np.array([[u for u in range(4) if u != v] for v in range(4)], np.uint32)
    idx = idx_with_graph(data, adj, 0)
    r = idx.search(np.array([[1.0]], np.float32), g.SearchParams(4, 2, 0.0))
    assert list(r.ids[0]) == [1, 2] and list(r.dists[0]) == [0.0, 0.0]


def test_start_override():  # test_search.cpp:167-180
    g = _g()
    data, adj = path_fixture(5)
    idx = idx_with_graph(data, adj, 4)
    q = np.array([[0.1]], np.float32)
    r = idx.search(q, g.SearchParams(5, 1, 0.0), start_override=[0])
    assert r.n_visited[0] == 1 and r.ids[0, 0] == 0
    r = idx.search(q, g.SearchParams(5, 1, 0.0), vcap=8)
    assert r.n_visited[0] == 5 and r.visited_ids[0, 0] == 4 and r.ids[0, 0] == 0


def test_validation():  # test_search.cpp:182-198
    g = _g()
    data, adj = path_fixture(3)
    idx = idx_with_graph(data, adj, 0)
    q = np.array([[1.0]], np.float32)
    for p in (g.SearchParams(2, 3, 0.0), g.SearchParams(2, 1, 0.3), g.SearchParams(0, 0, 0.0)):
        with pytest.raises(ValueError):
            idx.search(q, p)
    with pytest.raises(ValueError):
        idx.search(np.zeros((1, 2), np.float32), g.SearchParams(2, 1, 0.0))


@pytest.mark.parametrize("dtype", [np.uint8, np.int8])
@pytest.mark.parametrize("L,k,eps", [(10, 10, 0.0), (16, 10, 0.1), (50, 10, 0.25), (64, 64, 0.0),
                                     (128, 128, 0.0), (200, 200, 0.0), (4, 4, 0.0), (2, 1, 0.0)])
def test_search_parity_integer(oracle, dtype, L, k, eps):
    """Identical ids, distances, |V| and visit sequences over the reference's graph;
    REF visited mode also reproduces dist_comps."""
    g = _g()
    data, qs = mixture(11, 4000, 48, clusters=16, dtype=dtype, nq=300)
    adj, start = oracle.build(data, 24, 48, 1.2, workers=4)
    idx = idx_with_graph(data, adj, start)
    vcap = 4 * L + 64
    want = oracle.beam_search(adj, start, data, qs, L, k, eps, visited_mode=1, vcap=vcap, workers=4)
    for mode in ("fast", "ref"):
        got = idx.search(qs, g.SearchParams(L, k, eps), visited_mode=mode, vcap=vcap)
        assert (got.ids == want["ids"]).all()
        assert (got.dists == want["dists"]).all()
        assert (got.n_visited == want["n_visited"]).all()
        for i in range(len(qs)):
            nv = int(want["n_visited"][i])
            assert (got.visited_ids[i, :nv] == want["visited_ids"][i, :nv]).all()
            assert (got.visited_dists[i, :nv] == want["visited_dists"][i, :nv]).all()
        if mode == "ref":
            assert (got.dist_comps == want["dist_comps"]).all()


@pytest.mark.parametrize("L,k", [(10, 10), (64, 64), (128, 10)])
def test_exact_mode_counts_distinct_evaluations(oracle, orc, L, k):
    """EXACT visited mode: same ids/|V|, and dist_comps equals the restatement's
    exact seen-set count (the distinct-evaluation U of SURVEY.md §8d)."""
    g = _g()
    data, qs = mixture(13, 4000, 32, clusters=16, nq=200)
    adj, start = oracle.build(data, 24, 48, 1.2, workers=4)
    idx = idx_with_graph(data, adj, start)
    want = orc.beam_search(adj, start, data, qs, L, k, 0.0, visited_mode=0)
    got = idx.search(qs, g.SearchParams(L, k, 0.0), visited_mode="exact")
    assert (got.ids == want["ids"]).all() and (got.n_visited == want["n_visited"]).all()
    assert (got.dist_comps == want["dist_comps"]).all()
    fast = idx.search(qs, g.SearchParams(L, k, 0.0), visited_mode="fast")
    assert (fast.ids == want["ids"]).all() and (fast.dist_comps >= want["dist_comps"]).all()


@pytest.mark.parametrize("d", [16, 128, 256])
def test_search_parity_u8_widths(oracle, d):
    """Row widths exercise the 2/8/16-lanes-per-row gathers."""
    g = _g()
    data, qs = mixture(5, 3000, d, clusters=12, nq=200)
    adj, start = oracle.build(data, 32, 64, 1.2, workers=4)
    idx = idx_with_graph(data, adj, start)
    want = oracle.beam_search(adj, start, data, qs, 40, 40, 0.0, visited_mode=1, workers=4)
    got = idx.search(qs, g.SearchParams(40, 40, 0.0), visited_mode="ref")
    assert (got.ids == want["ids"]).all()
    assert (got.n_visited == want["n_visited"]).all()
    assert (got.dist_comps == want["dist_comps"]).all()


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_search_parity_f32(oracle, metric):
    """f32: same ids except where distances tie within 1e-5 relative (north star)."""
    g = _g()
    data, qs = mixture(9, 3000, 200 if metric == "ip" else 24, clusters=10, dtype=np.float32, nq=200)
    alpha = 1.0 if metric == "ip" else 1.2
    adj, start = oracle.build(data, 32, 64, alpha, metric=metric, workers=4)
    idx = idx_with_graph(data, adj, start, metric)
    want = oracle.beam_search(adj, start, data, qs, 32, 32, 0.0, metric=metric, workers=4)
    got = idx.search(qs, g.SearchParams(32, 32, 0.0))
    np.testing.assert_allclose(got.dists, want["dists"], rtol=1e-5, atol=1e-5)
    bad = 0
    for i in range(len(qs)):
        if not (got.ids[i] == want["ids"][i]).all():
            # every mismatch must be explained by a near-tie in distance
            d = np.sort(want["dists"][i])
            gaps = np.abs(np.diff(d)) <= 1e-5 * np.maximum(1.0, np.abs(d[1:]))
            assert gaps.any(), f"query {i}: ids differ without a distance tie"
            bad += 1
    assert bad <= len(qs) // 50


def test_search_k_out_prefix_of_gate(oracle):
    """Alg. 1 drained search {L, L, 0} reporting the top 10 (the primary sweep)."""
    g = _g()
    data, qs = mixture(21, 3000, 32, nq=100)
    adj, start = oracle.build(data, 24, 48, 1.2, workers=4)
    idx = idx_with_graph(data, adj, start)
    want = oracle.beam_search(adj, start, data, qs, 64, 64, 0.0, workers=4)
    got = idx.search(qs, g.SearchParams(64, 64, 0.0), k_out=10)
    assert (got.ids == want["ids"][:, :10]).all()
    with pytest.raises(ValueError):
        idx.search(qs, g.SearchParams(64, 10, 0.0), k_out=11)


def test_empty_and_single_point_graph(oracle):
    g = _g()
    data = np.array([[3, 4, 5, 6]], np.uint8)
    idx = g.Index(data, "l2", 4)
    idx.import_graph(np.full((1, 4), SENT, np.uint32), 0)
    r = idx.search(np.array([[0, 0, 0, 0]], np.uint8), g.SearchParams(4, 2, 0.0))
    assert r.ids[0, 0] == 0 and r.ids[0, 1] == SENT and r.n_visited[0] == 1
    assert r.dists[0, 0] == 9 + 16 + 25 + 36 and np.isinf(r.dists[0, 1])


def test_device_entry_matches_host_entry(oracle):
    torch = pytest.importorskip("torch")
    g = _g()
    data, qs = mixture(31, 2000, 128, nq=256)
    adj, start = oracle.build(data, 32, 64, 1.2, workers=4)
    idx = idx_with_graph(data, adj, start)
    host = idx.search(qs, g.SearchParams(32, 32, 0.0), k_out=10)
    tq = torch.from_numpy(qs).cuda()
    ids = torch.empty((len(qs), 10), dtype=torch.int32, device="cuda")
    dists = torch.empty((len(qs), 10), dtype=torch.float32, device="cuda")
    idx.search_device(tq.data_ptr(), len(qs), g.SearchParams(32, 32, 0.0), 10, ids.data_ptr(), dists.data_ptr(),
                      stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert (ids.cpu().numpy().view(np.uint32) == host.ids).all()
    idx.stage_queries(tq.data_ptr(), len(qs))
    ids.zero_()
    idx.search_staged(g.SearchParams(32, 32, 0.0), 10, ids.data_ptr(), dists.data_ptr(),
                      stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert (ids.cpu().numpy().view(np.uint32) == host.ids).all()


@pytest.mark.parametrize("dtype", [np.uint8, np.float32])
def test_search_async_concurrent_streams_equal_sync(dtype):
    """gann_search_async: batches enqueued on two streams (own scratch each,
    overlapping kernels) return exactly what the blocking gann_search does."""
    import torch
    g = _g()
    data, qs = mixture(71, 3000, 24, clusters=10, dtype=dtype, nq=700)
    idx = g.build_diskann(data, "l2", g.DiskannParams(16, 32, 1.2))
    sp = g.SearchParams(40, 10, 0.0)
    want = idx.search(qs, sp)
    qh = torch.from_numpy(np.ascontiguousarray(qs).view(np.uint8)).pin_memory()
    nq, k = qs.shape[0], 10
    streams = [torch.cuda.Stream() for _ in range(2)]
    nbytes = idx.async_scratch_bytes(nq, k)
    scratch = [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
    outs = [(torch.empty(nq * k, dtype=torch.int32).pin_memory(), torch.empty(nq * k, dtype=torch.float32).pin_memory())
            for _ in range(4)]
    for i, (oi, od) in enumerate(outs):
        s = streams[i % 2]
        idx.search_async(qh.data_ptr(), nq, sp, k, oi.data_ptr(), od.data_ptr(), scratch[i % 2].data_ptr(), nbytes,
                         s.cuda_stream)
    torch.cuda.synchronize()
    for oi, od in outs:
        assert (oi.numpy().view(np.uint32).reshape(nq, k) == want.ids).all()
        assert (od.numpy().reshape(nq, k) == want.dists).all()
    with pytest.raises(ValueError):
        idx.search_async(qh.data_ptr(), nq, sp, k, outs[0][0].data_ptr(), outs[0][1].data_ptr(),
                         scratch[0].data_ptr(), nbytes - 1, streams[0].cuda_stream)
    idx.close()


@pytest.mark.parametrize("env", [
    {"GANN_HASH_WAYS": "1"}, {"GANN_HASH_WAYS": "2"}, {"GANN_HASH_WAYS": "4"},
    {"GANN_HASH_WAYS": "4", "GANN_HASH_LOG2": "5"},   # 32 slots: constant evictions
    {"GANN_HASH_WAYS": "1", "GANN_HASH_LOG2": "5"},
    {"GANN_HASH16": "0"},                             # u32 id slots (4-way buckets)
    {"GANN_HASH16": "0", "GANN_HASH_LOG2": "5"},
    {"GANN_HASH16": "0", "GANN_HASH_WAYS": "1"},      # u32 id slots, direct mapped
    {"GANN_HASH16": "0", "GANN_HASH_WAYS": "1", "GANN_HASH_LOG2": "5"},
    {"GANN_SEARCH_DIAG": "1"},                        # general (diagnostic) kernel instance
])
def test_fast_filter_layouts_keep_results(oracle, monkeypatch, env):
    """The FAST visited table is a performance knob only: every layout (direct
    mapped or 2/4-way buckets of u16 remainders, u32 id slots, tiny tables that
    evict constantly) returns the reference's ids, distances, |V| and visit
    sequences; only the number of re-evaluations changes."""
    g = _g()
    data, qs = mixture(17, 4000, 48, clusters=16, nq=300)
    adj, start = oracle.build(data, 24, 48, 1.2, workers=4)
    idx = idx_with_graph(data, adj, start)
    L = 64
    vcap = 4 * L + 64
    want = oracle.beam_search(adj, start, data, qs, L, L, 0.0, visited_mode=1, vcap=vcap, workers=4)
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    got = idx.search(qs, g.SearchParams(L, L, 0.0), visited_mode="fast", vcap=vcap)
    assert (got.ids == want["ids"]).all()
    assert (got.dists == want["dists"]).all()
    assert (got.n_visited == want["n_visited"]).all()
    for i in range(len(qs)):
        nv = int(want["n_visited"][i])
        assert (got.visited_ids[i, :nv] == want["visited_ids"][i, :nv]).all()


def test_import_rejects_invalid_rows():
    """set_neighbors' checks (src/graph.cpp:42-59) and the distinct-neighbour
    invariant (check_graph_invariants, src/graph.cpp:80-92) at import; a
    failed import leaves an empty graph."""
    g = _g()
    data, adj = path_fixture(6)
    idx = g.Index(data, "l2", 2)
    for bad, msg in [((2, [1, 1]), "duplicate"), ((3, [3, 4]), "self loop"), ((4, [9, 5]), "out of range"),
                     ((5, [0xFFFFFFFF, 4]), "padding")]:
        a = adj.copy()
        a[bad[0]] = bad[1]
        with pytest.raises(ValueError, match=msg):
            idx.import_graph(a, 0)
        assert (idx.export_graph()[1] == 0).all()
    idx.import_graph(adj, 0)
    assert (idx.export_graph()[0] == adj).all()


def test_search_staged_needs_staged_queries():
    g = _g()
    data, adj = path_fixture(5)
    idx = idx_with_graph(data, adj, 0)
    with pytest.raises(ValueError, match="staged"):
        idx.search_staged(g.SearchParams(2, 1, 0.0), 1, 0, 0)
