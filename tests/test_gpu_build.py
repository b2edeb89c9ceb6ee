"""robustPrune, semisort, start vertex and full-build parity (CUDA vs CPU oracle).

Hand instances restate proj/tests/test_prune.cpp, test_semisort.cpp and
test_diskann.cpp; the randomized cases follow SURVEY.md §8c: prune bit-exact on
identical candidate lists, semisort equal to a stable sort by key, and the full
integer build bit-identical to the reference's build_diskann (uncapped) and to
its public-API capped loop."""
import numpy as np
import pytest

from helpers import degrees, mixture

pytestmark = pytest.mark.gpu
SENT = 0xFFFFFFFF


def _g():
    import paper_2305_04359_b200 as g
    return g


def l2_cands(data, p, ids):
    return [float(((data[p].astype(np.float64) - data[i]) ** 2).sum()) for i in ids]


def prune1(data, p, ids, R, alpha, rule="scale_candidate", metric="l2", dists=None):
    g = _g()
    idx = g.Index(np.ascontiguousarray(data), metric, R)
    d = l2_cands(data, p, ids) if dists is None else dists
    return list(g.alpha_prune(idx, p, ids, d, g.PruneParams(R, alpha, rule)))


def test_prune_single_candidate():  # test_prune.cpp:28-36
    assert prune1(np.array([[0], [5]], np.float32), 0, [1], 64, 1.2) == [1]


def test_prune_alpha_on_the_line():  # test_prune.cpp:38-56
    data = np.array([[0], [1], [2], [4]], np.float32)
    assert prune1(data, 0, [1, 2, 3], 3, 1.0) == [1]
    assert prune1(data, 0, [1, 2, 3], 3, 2.0) == [1, 3]


def test_prune_rules_disagree():  # test_prune.cpp:58-76
    data = np.array([[0.0], [1.0], [1.9]], np.float32)
    assert prune1(data, 0, [1, 2], 3, 0.5, "scale_candidate") == [1]
    assert prune1(data, 0, [1, 2], 3, 0.5, "scale_selected") == [1, 2]


def test_prune_zero_distance_twins():  # test_prune.cpp:78-91
    data = np.array([[0], [0], [0], [1], [2]], np.float32)
    assert prune1(data, 0, [1, 2, 3, 4], 8, 1.0) == [1, 2, 3]


def test_prune_skips_p_and_caps_at_R():  # test_prune.cpp:93-105
    data = np.array([[0], [1], [10], [20], [30]], np.float32)
    out = prune1(data, 0, [0, 1, 2, 3, 4], 2, 2.0)
    assert len(out) == 2 and out[0] == 1 and 0 not in out


@pytest.mark.parametrize("dtype", [np.uint8, np.int8, np.float32])
@pytest.mark.parametrize("rule", ["scale_candidate", "scale_selected"])
@pytest.mark.parametrize("alpha", [0.8, 1.0, 1.2, 2.0])
def test_prune_parity_on_reference_visited_lists(oracle, dtype, rule, alpha):
    """alpha_prune on the reference's own insert-time candidate lists (its
    visited sets) is bit-exact against the reference."""
    g = _g()
    data, qs = mixture(3, 3000, 32, clusters=10, dtype=dtype, nq=200)
    adj, start = oracle.build(data, 32, 64, 1.2, workers=4)
    vis = oracle.beam_search(adj, start, data, data[:200], 64, 64, vcap=256, workers=4)
    R = 16
    idx = g.Index(data, "l2", R)
    lists, dl, ps = [], [], []
    for i in range(200):
        nv = int(vis["n_visited"][i])
        lists.append(vis["visited_ids"][i, :nv])
        dl.append(vis["visited_dists"][i, :nv])
        ps.append(i)
    got = idx.alpha_prune_many(ps, lists, dl, g.PruneParams(R, alpha, rule))
    for i in range(200):
        want, _ = oracle.alpha_prune(ps[i], lists[i], dl[i], data, R, alpha, rule)
        assert list(got[i]) == list(want), f"list {i}"


@pytest.mark.parametrize("alpha,R", [(1.2, 64), (0.5, 64), (0.8, 16), (2.0, 8)])
def test_prune_parity_long_lists(oracle, alpha, R):
    """Hub-sized lists (the chunked path, several 4096-key chunks when the
    selections run out) are bit-exact too."""
    g = _g()
    data = mixture(4, 30000, 16, clusters=4)
    rng = np.random.default_rng(0)
    idx = g.Index(data, "l2", R)
    ps, lists, dl = [], [], []
    for m in (513, 600, 2000, 9000, 25000):
        p = int(rng.integers(0, len(data)))
        ids = rng.choice(len(data), m, replace=False).astype(np.uint32)
        ps.append(p)
        lists.append(ids)
        dl.append(np.array(l2_cands(data, p, ids), np.float32))
    got = idx.alpha_prune_many(ps, lists, dl, g.PruneParams(R, alpha))
    for i in range(len(ps)):
        want, _ = oracle.alpha_prune(ps[i], lists[i], dl[i], data, R, alpha)
        assert list(got[i]) == list(want), f"list {i} (m={len(lists[i])})"


def _check_grouping(keys, vals, got):
    """Sort-based oracle of test_semisort.cpp:19-53."""
    assert len(got.keys) == len(keys)
    assert sorted(zip(got.keys.tolist(), got.vals.tolist())) == sorted(zip(keys.tolist(), vals.tolist()))
    off = got.group_offsets.astype(np.int64)
    if len(keys) == 0:
        assert got.groups() == 0
        return
    assert off[0] == 0 and off[-1] == len(keys)
    seen = set()
    for gi in range(got.groups()):
        lo, hi = off[gi], off[gi + 1]
        assert lo < hi
        k = got.keys[lo]
        assert k not in seen
        seen.add(k)
        assert (got.keys[lo:hi] == k).all()
        assert (got.vals[lo:hi] == vals[keys == k]).all()  # input order within the group
    assert len(seen) == len(set(keys.tolist()))


def test_group_by_key_many_seeds():  # test_semisort.cpp:57-70
    g = _g()
    for seed in range(30):
        rng = np.random.default_rng(seed)
        n = int(1 + rng.integers(0, 3000))
        space = int(1 + rng.integers(0, 200))
        keys = rng.integers(0, space, n).astype(np.uint32)
        vals = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
        _check_grouping(keys, vals, g.group_by_key(keys, vals))


def test_group_by_key_edge_shapes():  # test_semisort.cpp:87-113
    g = _g()
    e = g.group_by_key(np.zeros(0, np.uint32), np.zeros(0, np.uint32))
    assert e.groups() == 0 and len(e.keys) == 0
    k = np.full(100, 3, np.uint32)
    v = np.arange(100, dtype=np.uint32)
    got = g.group_by_key(k, v)
    assert got.groups() == 1 and (got.vals == v).all()
    k = np.arange(64, dtype=np.uint32)
    _check_grouping(k, k * 2, g.group_by_key(k, k * 2))
    k = (np.arange(4096, dtype=np.uint32) << 20).astype(np.uint32)
    _check_grouping(k, np.arange(4096, dtype=np.uint32), g.group_by_key(k, np.arange(4096, dtype=np.uint32)))


def test_group_by_key_matches_reference_groups(oracle):
    """Acceptance criterion 10 shape (tests/acceptance.cpp:538-597): 100k pairs."""
    g = _g()
    for seed in range(5):
        rng = np.random.default_rng(100 + seed)
        keys = rng.integers(0, 5000, 100_000).astype(np.uint32)
        vals = rng.integers(0, 2**32, 100_000, dtype=np.uint64).astype(np.uint32)
        got = g.group_by_key(keys, vals)
        ok, ov, off = oracle.group_by_key(keys, vals)
        ref = {int(ok[off[i]]): ov[off[i]:off[i + 1]].tolist() for i in range(len(off) - 1)}
        mine = {int(got.keys[got.group_offsets[i]]): got.vals[got.group_offsets[i]:got.group_offsets[i + 1]].tolist()
                for i in range(got.groups())}
        assert mine == ref


@pytest.mark.parametrize("dtype,metric", [(np.uint8, "l2"), (np.int8, "l2"), (np.uint8, "ip"), (np.float32, "l2")])
def test_choose_start(oracle, dtype, metric):  # test_diskann.cpp:32-66
    g = _g()
    data = mixture(8, 5000, 40, dtype=dtype)
    idx = g.Index(data, metric, 8)
    assert idx.choose_start() == oracle.choose_start(data, metric)


def test_choose_start_hand():
    g = _g()
    assert g.Index(np.array([[0, 0], [10, 10]], np.float32), "l2", 2).choose_start() == 0
    assert g.Index(np.array([[0, 0], [0, 0], [9, 9]], np.float32), "l2", 2).choose_start() == 0
    assert g.Index(np.array([[4, 4]], np.float32), "l2", 2).choose_start() == 0


def test_insert_into_start_only_graph():  # test_diskann.cpp:79-104
    g = _g()
    data = np.array([[0], [3], [7]], np.float32)
    idx = g.Index(data, "l2", 2)
    idx.import_graph(np.full((3, 2), SENT, np.uint32), 0)
    assert g.insert_point(idx, 1, 4, 1.2) == [(0, 1)]
    adj, _, _ = idx.export_graph()
    assert list(adj[1]) == [0, SENT]
    adj[0] = [1, SENT]
    idx.import_graph(adj, 0)
    assert g.insert_point(idx, 2, 4, 1.2) == [(1, 2)]
    adj, _, _ = idx.export_graph()
    assert list(adj[2]) == [1, SENT]


def test_apply_back_edges_parity(oracle):
    """Phase 2 alone on explicit pairs (duplicates and hubs included)."""
    g = _g()
    data = mixture(12, 3000, 32)
    adj, start = oracle.build(data, 16, 32, 1.2, workers=4)
    rng = np.random.default_rng(5)
    t = rng.integers(0, 3000, 20000).astype(np.uint32)
    t[:3000] = 7  # a hub
    s = rng.integers(0, 3000, 20000).astype(np.uint32)
    keep = t != s
    t, s = t[keep], s[keep]
    want = oracle.apply_back_edges(adj, data, t, s, 1.2, workers=4)
    idx = g.Index(data, "l2", 16)
    idx.import_graph(adj, start)
    idx.apply_back_edges(t, s, g.PruneParams(16, 1.2))
    got, _, _ = idx.export_graph()
    assert (got == want).all()


@pytest.mark.parametrize("alpha,rule", [(1.0, "scale_candidate"), (1.2, "scale_selected"), (1.2, "scale_candidate")])
def test_apply_back_edges_after_gpu_build(oracle, alpha, rule):
    """Re-prunes of rows the GPU build wrote (their prune prefixes are known to
    be mutually non-culling under the build's alpha/rule): with the same
    parameters the prefix pairs are skipped, with other ones they are not.
    Either way the result is the reference's apply_back_edges."""
    g = _g()
    data = mixture(13, 3000, 32, clusters=12)
    idx = g.build_diskann(data, "l2", g.DiskannParams(16, 32, 1.2))
    adj, _, start = idx.export_graph()
    rng = np.random.default_rng(9)
    t = rng.integers(0, 3000, 12000).astype(np.uint32)
    s = rng.integers(0, 3000, 12000).astype(np.uint32)
    keep = t != s
    t, s = t[keep], s[keep]
    want = oracle.apply_back_edges(adj, data, t, s, alpha, rule=rule, workers=4)
    idx.apply_back_edges(t, s, g.PruneParams(16, alpha, rule))
    got, _, _ = idx.export_graph()
    assert (got == want).all(), f"{int((got != want).any(axis=1).sum())} rows differ"
    # and once more on top (prefixes now from these re-prunes)
    want2 = oracle.apply_back_edges(want, data, s, t, alpha, rule=rule, workers=4)
    idx.apply_back_edges(s, t, g.PruneParams(16, alpha, rule))
    got2, _, _ = idx.export_graph()
    assert (got2 == want2).all()
    idx.close()


@pytest.mark.parametrize("dtype", [np.uint8, np.int8])
@pytest.mark.parametrize("cap", [0, 97])
def test_build_bit_identical(oracle, dtype, cap):
    """Integer build == the reference's build (uncapped: build_diskann itself)."""
    g = _g()
    data = mixture(17, 6000, 32, clusters=20, dtype=dtype)
    want, ws = oracle.build(data, 24, 48, 1.2, cap=cap, workers=8)
    idx = g.build_diskann(data, "l2", g.DiskannParams(24, 48, 1.2, max_batch=cap))
    got, deg, s = idx.export_graph()
    assert s == ws
    assert (deg == degrees(want)).all()
    assert (got == want).all()


@pytest.mark.parametrize("d,dtype,metric", [(128, np.uint8, "l2"), (256, np.uint8, "l2"), (48, np.int8, "l2"),
                                            (128, np.uint8, "ip")])
def test_build_bit_identical_widths(oracle, d, dtype, metric):
    """Wider rows (the tensor-core prune's 4 and 8 k-steps, a 16-byte tail at d=48)."""
    g = _g()
    data = mixture(29, 4000, d, clusters=12, dtype=dtype)
    want, ws = oracle.build(data, 32, 64, 1.2, metric=metric, workers=8)
    idx = g.build_diskann(data, metric, g.DiskannParams(32, 64, 1.2))
    got, _, s = idx.export_graph()
    assert s == ws and (got == want).all()


def test_build_long_walk_rerun(oracle, monkeypatch):
    """Inserts whose visited list outgrows the buffer are re-searched exactly
    (forced here with a tiny buffer): the graph stays bit-identical."""
    g = _g()
    data = mixture(23, 3000, 32, clusters=10)
    want, ws = oracle.build(data, 16, 32, 1.2, workers=8)
    monkeypatch.setenv("GANN_VCAP", "8")
    idx = g.build_diskann(data, "l2", g.DiskannParams(16, 32, 1.2))
    got, _, s = idx.export_graph()
    assert s == ws and (got == want).all()


def test_build_bit_identical_ip_and_selected_rule(oracle):
    g = _g()
    data = mixture(18, 4000, 24, clusters=10)
    want, ws = oracle.build(data, 16, 32, 0.9, rule="scale_selected", metric="ip", workers=8)
    idx = g.build_diskann(data, "ip", g.DiskannParams(16, 32, 0.9, rule="scale_selected"))
    got, _, s = idx.export_graph()
    assert s == ws and (got == want).all()


def test_build_f32_recall_within_half_point(oracle):
    """f32 (FMA partial sums on the GPU): recall@10 within 0.5 points of the reference graph."""
    g = _g()
    data, qs = mixture(19, 6000, 16, clusters=8, dtype=np.float32, nq=500)
    want, ws = oracle.build(data, 24, 48, 1.2, workers=8)
    idx = g.build_diskann(data, "l2", g.DiskannParams(24, 48, 1.2))
    got, _, s = idx.export_graph()
    gt_ids, gt_d = oracle.groundtruth(data, qs, 10)
    r_ref = oracle.beam_search(want, ws, data, qs, 10, 10, workers=8)
    r_gpu = idx.search(qs, g.SearchParams(10, 10, 0.0))
    rec_ref = oracle.mean_recall(gt_ids, gt_d, r_ref["ids"], 10)
    rec_gpu = oracle.mean_recall(gt_ids, gt_d, r_gpu.ids, 10)
    assert rec_gpu >= rec_ref - 0.005, (rec_gpu, rec_ref)


def test_build_invariants_and_degenerate():  # test_diskann.cpp:106-120, 179-196
    g = _g()
    data = mixture(33, 2000, 8, clusters=5, dtype=np.float32)
    idx = g.build_diskann(data, "l2", g.DiskannParams(16, 32, 1.2))
    adj, deg, s = idx.export_graph()
    assert deg.max() <= 16 and deg.mean() > 2.0
    for v in range(len(adj)):
        row = adj[v, : deg[v]]
        assert len(set(row.tolist())) == len(row) and v not in row and (row < 2000).all()
        assert (adj[v, deg[v]:] == SENT).all()
    one = g.build_diskann(np.array([[1, 2]], np.float32), "l2", g.DiskannParams())
    assert one.export_graph()[1].sum() == 0
    same = g.build_diskann(np.full((10, 2), 3.0, np.float32), "l2", g.DiskannParams(4, 8, 1.2))
    a, d, _ = same.export_graph()
    for v in range(10):
        assert v not in a[v, : d[v]]
    with pytest.raises(ValueError):
        g.build_diskann(np.zeros((0, 4), np.uint8), "l2", g.DiskannParams())


def test_alpha_thickens_graph():  # test_diskann.cpp:122-135
    g = _g()
    data = mixture(34, 1500, 8, clusters=5, dtype=np.float32)
    prev = 0.0
    for alpha in (1.0, 1.1, 1.2):
        deg = g.build_diskann(data, "l2", g.DiskannParams(16, 32, alpha)).export_graph()[1]
        assert deg.mean() >= prev
        prev = deg.mean()


def test_groundtruth_parity(oracle):
    g = _g()
    data, qs = mixture(41, 20000, 128, clusters=50, nq=300)
    idx = g.Index(data, "l2", 8)
    ids, dists = idx.groundtruth(qs, 10)
    wi, wd = oracle.groundtruth(data, qs, 10)
    assert (ids == wi).all() and (dists == wd).all()


def test_generator_matches_numpy_restatement():
    torch = pytest.importorskip("torch")
    from paper_2305_04359_b200 import datagen
    from paper_2305_04359_b200._lib import check, lib
    for (n, d, cl, sig, nf) in [(3000, 128, 1000, 20.0, 0.0), (2000, 256, 5000, 12.0, 0.1)]:
        buf = torch.empty(n * d, dtype=torch.uint8, device="cuda")
        check(lib().gann_generate_u8(buf.data_ptr(), n, d, cl, sig, nf, 1, 2, 500, 0))
        want = datagen.gen_u8_numpy(n, d, cl, sig, nf, 1, 2, row0=500)
        assert (buf.cpu().numpy().reshape(n, d) == want).all()


def test_f32_generator_matches_numpy_restatement():
    """Config 3's generator: device rows equal the float64 restatement after
    the one f32 rounding (tolerance: the warp-order sum of squares)."""
    torch = pytest.importorskip("torch")
    from paper_2305_04359_b200 import datagen
    from paper_2305_04359_b200._lib import check, lib
    for (n, d, cl, sig, ns, sh) in [(3000, 200, 2000, 0.5, 0.3, 0.0), (1000, 200, 2000, 0.5, 0.3, 0.5),
                                    (500, 37, 7, 1.0, 0.0, 0.0)]:
        buf = torch.empty(n * d, dtype=torch.float32, device="cuda")
        check(lib().gann_generate_f32(buf.data_ptr(), n, d, cl, sig, ns, sh, 1, 2, 700, 0))
        want = datagen.gen_f32_numpy(n, d, cl, sig, ns, sh, 1, 2, row0=700)
        got = buf.cpu().numpy().reshape(n, d)
        np.testing.assert_allclose(got, want, rtol=2e-6, atol=1e-7)
        assert (got == want).mean() > 0.99


def test_cpp_dropin_runs():
    """The reference's hand instances through include/gann.hpp (C++)."""
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    subprocess.run(["make", "-s", "-C", str(root / "tests" / "cpp")], check=True)
    r = subprocess.run([str(root / "tests" / "cpp" / "_build" / "test_gann_cpp")], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stderr
    assert "ok" in r.stdout


def test_build_long_walks_beyond_every_bin(oracle, monkeypatch):
    """Walks longer than both the visited buffer and the largest prune bin
    (|V| > max(vcap, 512), the chunked kernel's range) are skipped by the
    first prune pass and re-run: the graph stays bit-identical."""
    g = _g()
    data = mixture(24, 3000, 16, clusters=10)
    want, ws = oracle.build(data, 16, 600, 1.2, workers=8)
    monkeypatch.setenv("GANN_VCAP", "64")
    idx = g.build_diskann(data, "l2", g.DiskannParams(16, 600, 1.2))
    got, _, s = idx.export_graph()
    assert s == ws and (got == want).all()


def test_alpha_prune_rejects_repeated_candidates():
    """A candidate list repeating an id is rejected (the kernels' rank sort
    needs distinct keys); copies of p itself are dropped as in prune.cpp:16-18."""
    g = _g()
    data = mixture(25, 200, 8, clusters=3)
    idx = g.Index(data, "l2", 8)
    p = g.PruneParams(8, 1.2)
    ids = np.array([3, 4, 5, 4], np.uint32)
    with pytest.raises(ValueError, match="repeats"):
        idx.alpha_prune_many([0], [ids], [np.array(l2_cands(data, 0, ids), np.float32)], p)
    ids = np.array([0, 3, 0, 4], np.uint32)  # p twice: fine
    got = idx.alpha_prune_many([0], [ids], [np.array(l2_cands(data, 0, ids), np.float32)], p)
    assert 0 not in list(got[0])
