"""Parity at the BASELINE parameters (R=64, L=128/200, alpha=1.2).

SURVEY.md §8c's protocol at the shape every benchmarked config uses:

* config 0 exactly (datagen c0: 100k x 128 u8, 1000 clusters, sigma 20;
  R64 L128 alpha 1.2), uncapped and with the config's 2% batch cap: the GPU
  graph and start vertex are bit-identical to graphann's (build_diskann,
  src/diskann.cpp:31-70, and its public-API capped loop);
* beam search over graphann's own c0 graph (src/search.cpp:62-131) at
  {L, L, 0} for L in 10..200 and at the reference eval semantics {L, 10, eps}:
  ids, distances, |V| and visit sequences identical, and in REF visited mode
  dist_comps identical too — rows of 64 ids use both adjacency registers;
* alpha_prune (src/prune.cpp:8-44) at R=64 on graphann's own visited lists of
  L=128/200/300 walks: lists of 129-512 candidates, i.e. the W=8/16
  tensor-core bins of the c1 insert regime (|V| ~ 1.3 L at 10M);
* d=256 (config 2's generator, 16-lane rows): bit-identical R64 build and
  search parity through both compile-time degree instances (GANN_SEARCH_R64=1
  and =0).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NQ = 2000


def _g():
    import paper_2305_04359_b200 as g
    return g


@pytest.fixture(scope="module")
def c0():
    from paper_2305_04359_b200 import datagen
    cfg = datagen.CONFIGS["c0"]
    return cfg, datagen.host_base(cfg), datagen.host_queries(cfg, NQ)


@pytest.fixture(scope="module")
def c0_ref(oracle, c0):
    """graphann's uncapped build_diskann graph of config 0."""
    cfg, data, _ = c0
    return oracle.build(data, cfg.R, cfg.L, cfg.alpha, cap=0, workers=0)


@pytest.fixture(scope="module")
def c0_index(c0, c0_ref):
    g = _g()
    cfg, data, _ = c0
    adj, start = c0_ref
    idx = g.Index(data, "l2", cfg.R)
    idx.import_graph(adj, start)
    return idx


@pytest.mark.parametrize("capped", [False, True])
def test_c0_build_bit_identical(oracle, c0, c0_ref, capped):
    g = _g()
    cfg, data, _ = c0
    cap = cfg.max_batch if capped else 0
    assert not capped or cap == 2000
    want, ws = c0_ref if not capped else oracle.build(data, cfg.R, cfg.L, cfg.alpha, cap=cap, workers=0)
    idx = g.build_diskann(data, "l2", g.DiskannParams(cfg.R, cfg.L, cfg.alpha, max_batch=cap))
    got, deg, s = idx.export_graph()
    assert s == ws
    assert (deg == (want != 0xFFFFFFFF).sum(1)).all()
    bad = np.nonzero((got != want).any(axis=1))[0]
    assert len(bad) == 0, f"{len(bad)} of {len(want)} rows differ (first {bad[:5].tolist()})"
    assert deg.max() == 64  # full rows: the second adjacency register is exercised


def _check_search(got, want, check_dc):
    assert (got.ids == want["ids"]).all()
    assert (got.dists == want["dists"]).all()
    assert (got.n_visited == want["n_visited"]).all()
    nv = want["n_visited"].astype(np.int64)
    pos = np.arange(want["visited_ids"].shape[1])[None, :] < nv[:, None]
    assert (got.visited_ids[pos] == want["visited_ids"][pos]).all()
    assert (got.visited_dists[pos] == want["visited_dists"][pos]).all()
    if check_dc:
        assert (got.dist_comps == want["dist_comps"]).all()


@pytest.mark.parametrize("L", [10, 64, 128, 200])
def test_c0_search_parity_alg1(oracle, c0, c0_ref, c0_index, L):
    """{L, L, 0} (Alg. 1, the build's own search) over graphann's c0 graph."""
    g = _g()
    _, data, qs = c0
    adj, start = c0_ref
    vcap = 2 * L + 64
    want = oracle.beam_search(adj, start, data, qs, L, L, 0.0, visited_mode=1, vcap=vcap, workers=0)
    assert want["n_visited"].max() <= vcap
    for mode in ("fast", "ref"):
        got = c0_index.search(qs, g.SearchParams(L, L, 0.0), visited_mode=mode, vcap=vcap)
        _check_search(got, want, mode == "ref")


@pytest.mark.parametrize("L", [16, 64, 128, 200])
@pytest.mark.parametrize("eps", [0.0, 0.1, 0.25])
def test_c0_search_parity_eval_semantics(oracle, c0, c0_ref, c0_index, L, eps):
    """The reference eval's {L, 10, eps} (src/eval.cpp:151-153), top-10."""
    g = _g()
    _, data, qs = c0
    adj, start = c0_ref
    vcap = 2 * L + 64
    want = oracle.beam_search(adj, start, data, qs, L, 10, eps, visited_mode=1, vcap=vcap, workers=0)
    got = c0_index.search(qs, g.SearchParams(L, 10, eps), visited_mode="ref", vcap=vcap)
    _check_search(got, want, True)


@pytest.mark.parametrize("L", [128, 200, 300])
@pytest.mark.parametrize("rule", ["scale_candidate", "scale_selected"])
def test_c0_prune_parity_R64(oracle, c0, c0_ref, c0_index, L, rule):
    """alpha_prune at R=64 on graphann's own insert-style visited lists (the
    walk from a data point itself, as insert_point does)."""
    _, data, _ = c0
    adj, start = c0_ref
    rows = np.arange(0, len(data), len(data) // 1500, dtype=np.int64)[:1500]
    vcap = 3 * L
    vis = oracle.beam_search(adj, start, data, data[rows], L, L, 0.0, vcap=vcap, workers=0)
    nv = vis["n_visited"].astype(np.int64)
    assert nv.max() <= vcap
    assert (nv > 128).mean() > 0.5  # the W=8 bin (129-256 candidates; at c0 |V| ~ L)
    if L == 300:
        assert (nv > 256).mean() > 0.5  # ... and the W=16 bin (257-512)
    ps = rows.astype(np.uint32).tolist()
    lists = [vis["visited_ids"][i, :nv[i]] for i in range(len(rows))]
    dl = [vis["visited_dists"][i, :nv[i]] for i in range(len(rows))]
    got = c0_index.alpha_prune_many(ps, lists, dl, _g().PruneParams(64, 1.2, rule))
    for i in range(len(rows)):
        want, _ = oracle.alpha_prune(ps[i], lists[i], dl[i], data, 64, 1.2, rule)
        assert list(got[i]) == list(want), f"list {i} (|V| = {nv[i]})"


@pytest.fixture(scope="module")
def c2_small(oracle):
    """Config 2's generator (d=256, 5000 clusters, sigma 12, 10% noise) at 40k
    points, with graphann's uncapped R64 L128 graph."""
    from paper_2305_04359_b200 import datagen
    cfg = datagen.CONFIGS["c2"].scaled(40_000)
    data, qs = datagen.host_base(cfg), datagen.host_queries(cfg, 1000)
    adj, start = oracle.build(data, cfg.R, cfg.L, cfg.alpha, cap=0, workers=0)
    return cfg, data, qs, adj, start


def test_c2_build_bit_identical_d256(c2_small):
    g = _g()
    cfg, data, _, want, ws = c2_small
    idx = g.build_diskann(data, "l2", g.DiskannParams(cfg.R, cfg.L, cfg.alpha))
    got, deg, s = idx.export_graph()
    assert s == ws
    bad = np.nonzero((got != want).any(axis=1))[0]
    assert len(bad) == 0, f"{len(bad)} rows differ"


@pytest.mark.parametrize("r64", ["1", "0"])
@pytest.mark.parametrize("L,k", [(128, 128), (200, 200), (128, 10)])
def test_c2_search_parity_d256_R64(oracle, c2_small, monkeypatch, r64, L, k):
    """16-lane rows at R=64: the compile-time R64 instance and the generic one."""
    g = _g()
    cfg, data, qs, adj, start = c2_small
    idx = g.Index(data, "l2", cfg.R)
    idx.import_graph(adj, start)
    vcap = 2 * L + 64
    want = oracle.beam_search(adj, start, data, qs, L, k, 0.0, visited_mode=1, vcap=vcap, workers=0)
    monkeypatch.setenv("GANN_SEARCH_R64", r64)
    got = idx.search(qs, g.SearchParams(L, k, 0.0), visited_mode="fast", vcap=vcap)
    _check_search(got, want, False)
