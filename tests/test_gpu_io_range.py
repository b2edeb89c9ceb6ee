"""Graph / dataset files in the reference's formats and range search
(SURVEY.md §8f rows 2-3), checked against the reference's own code."""
import numpy as np
import pytest

from helpers import mixture

pytestmark = pytest.mark.gpu
SENT = 0xFFFFFFFF


def _g():
    import paper_2305_04359_b200 as g
    return g


def test_anng_roundtrip_with_reference(oracle, tmp_path):
    """A GPU-built graph saved as ANNG loads in graphann (load_graph), and a
    graph saved by graphann loads into the index — byte-identical files."""
    g = _g()
    data = mixture(51, 3000, 32, clusters=10)
    idx = g.build_diskann(data, "l2", g.DiskannParams(16, 32, 1.2))
    adj, _, start = idx.export_graph()
    idx.save_graph(tmp_path / "gpu.anng")
    radj, rstart = oracle.load_graph(tmp_path / "gpu.anng")
    assert rstart == start and (radj == adj).all()
    oracle.save_graph(adj, start, tmp_path / "ref.anng")
    assert (tmp_path / "gpu.anng").read_bytes() == (tmp_path / "ref.anng").read_bytes()
    idx2 = g.Index(data, "l2", 16)
    idx2.load_graph(tmp_path / "ref.anng")
    a2, _, s2 = idx2.export_graph()
    assert s2 == start and (a2 == adj).all()


def test_anng_rejects_malformed_files(tmp_path):
    g = _g()
    data = mixture(52, 100, 8)
    idx = g.Index(data, "l2", 8)
    (tmp_path / "bad.anng").write_bytes(b"NOPE" + b"\0" * 32)
    with pytest.raises(IOError):
        idx.load_graph(tmp_path / "bad.anng")
    good = g.build_diskann(data, "l2", g.DiskannParams(8, 16, 1.2))
    good.save_graph(tmp_path / "g.anng")
    raw = (tmp_path / "g.anng").read_bytes()
    (tmp_path / "trunc.anng").write_bytes(raw[:-4])
    with pytest.raises(IOError):
        idx.load_graph(tmp_path / "trunc.anng")
    (tmp_path / "trail.anng").write_bytes(raw + b"\0\0\0\0")
    with pytest.raises(IOError):
        idx.load_graph(tmp_path / "trail.anng")
    with pytest.raises(IOError):
        idx.load_graph(tmp_path / "missing.anng")


@pytest.mark.parametrize("ext,dtype,fmt", [("u8bin", np.uint8, "bin"), ("i8bin", np.int8, "bin"),
                                            ("fbin", np.float32, "bin"), ("bvecs", np.uint8, "vecs"),
                                            ("fvecs", np.float32, "vecs")])
def test_vectors_written_by_reference_load(oracle, tmp_path, ext, dtype, fmt):
    g = _g()
    data, qs = mixture(53, 800, 24, dtype=dtype, nq=20)
    path = tmp_path / f"x.{ext}"
    oracle.write_vectors(data, path, fmt)
    a = g.Index.from_file(str(path), "l2", 12)
    b = g.Index(data, "l2", 12)
    assert a.n == 800 and a.d == 24 and a.dtype == np.dtype(dtype)
    a.build(g.DiskannParams(12, 24, 1.2))
    b.build(g.DiskannParams(12, 24, 1.2))
    assert (a.export_graph()[0] == b.export_graph()[0]).all()


def test_range_search_matches_reference(oracle):  # test_search.cpp:223-238 + random
    g = _g()
    data, qs = mixture(54, 3000, 16, clusters=10, nq=60)
    adj, start = oracle.build(data, 16, 32, 1.2, workers=4)
    idx = g.Index(data, "l2", 16)
    idx.import_graph(adj, start)
    for radius, L, eps in [(90.0, 32, 0.0), (110.0, 64, 0.1), (70.0, 16, 0.0)]:
        got = idx.range_search(qs, radius, g.SearchParams(L, 1, eps))
        want, counts = oracle.range_search(adj, start, data, qs, radius, L, eps, cap=4096)
        for i in range(len(qs)):
            assert (got[i][0] == want[i][0]).all() and (got[i][1] == want[i][1]).all(), (radius, i)
        assert sum(len(x[0]) for x in got) > 0


def test_range_search_hand_instance():
    g = _g()
    data = np.arange(5, dtype=np.float32).reshape(5, 1)
    adj = np.full((5, 2), SENT, np.uint32)
    for i in range(5):
        nb = ([i - 1] if i > 0 else []) + ([i + 1] if i + 1 < 5 else [])
        adj[i, : len(nb)] = nb
    idx = g.Index(data, "l2", 2)
    idx.import_graph(adj, 0)
    (ids, dists), = idx.range_search(np.array([[2.2]], np.float32), 1.3, g.SearchParams(5, 1, 0.0))
    assert list(ids) == [2, 3, 1]
    with pytest.raises(ValueError):
        idx.range_search(np.array([[2.2]], np.float32), -1.0, g.SearchParams(5, 1, 0.0))
