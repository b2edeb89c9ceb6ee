"""CPU: the C-ABI library loads and exports include/gann.h; host-side schedule
helpers match the reference; the numpy data generator and recall scoring."""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _lib():
    from paper_2305_04359_b200._lib import LIB_PATH, lib
    if not LIB_PATH.exists():
        pytest.fail(f"{LIB_PATH} not built (run __graft_entry__.build())")
    return lib()


def test_library_exports_every_header_symbol():
    import ctypes
    header = (ROOT / "include" / "gann.h").read_text()
    decls = set(re.findall(r"\b(gann_[a-z_0-9]+)\s*\(", header))
    assert len(decls) >= 25
    L = _lib()
    missing = [d for d in sorted(decls) if not hasattr(L, d)]
    assert not missing, missing
    from paper_2305_04359_b200._lib import SIGNATURES
    assert set(SIGNATURES) == decls, set(SIGNATURES) ^ decls
    assert L.gann_version().decode().endswith("sm_100a")
    assert isinstance(L.gann_last_error(), bytes)
    del ctypes


def test_library_is_sm100a_code():
    import subprocess
    from paper_2305_04359_b200._lib import LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_means_loud_failure():
    """Without a GPU every compute entry point fails with an error (never a CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2305_04359_b200 as g
    with pytest.raises(g.GannError):
        g.Index(np.zeros((4, 8), np.uint8), "l2", 4)


def test_host_schedule_matches_reference(orc):
    import paper_2305_04359_b200 as g
    for n, cap in [(10, 0), (1, 0), (2, 0), (3, 0), (1000, 0), (100000, 2000), (10_000_000, 200_000)]:
        assert g.batch_ranges(n, cap) == orc.batch_ranges(n, cap)
    assert (g.shuffled_order(1000, 42, 17) == orc.shuffled_order(1000, 42, 17)).all()
    assert g.insert_seed(42) == 16503569613174706033


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 1000, 1001, 65536, 300_001])
def test_shuffle_swap_log_replays_to_the_reference_order(orc, n):
    """gann_build draws std::shuffle's swap log on the host (the same libstdc++
    call over a logging iterator) and resolves the permutation on the device;
    here the log is replayed sequentially and must give shuffled_order
    (src/builder_common.cpp:99-107) before its front swap — odd and even n
    (libstdc++ pairs the swaps and does an extra first one for even n)."""
    import paper_2305_04359_b200 as g
    seed = g.insert_seed(42)
    log = g.shuffle_swap_log(n, seed)
    assert log[0] == 0 and (log <= np.arange(n)).all()
    a = list(range(n))
    for i in range(1, n):
        j = int(log[i])
        a[i], a[j] = a[j], a[i]
    want = orc.shuffled_order(n, seed, a[0])  # front = the element already first: no front swap
    assert (np.array(a, np.uint32) == want).all()


def test_datagen_is_deterministic_and_prefix_stable():
    from paper_2305_04359_b200 import datagen
    a = datagen.gen_u8_numpy(500, 128, 1000, 20.0, 0.0, 1, 2)
    b = datagen.gen_u8_numpy(300, 128, 1000, 20.0, 0.0, 1, 2, row0=200)
    assert (a[200:] == b).all()
    assert (a == datagen.gen_u8_numpy(500, 128, 1000, 20.0, 0.0, 1, 2)).all()
    assert not (a == datagen.gen_u8_numpy(500, 128, 1000, 20.0, 0.0, 1, 3)).all()


def test_normal_table_pinned_to_library():
    """The generators' Gaussian quantile table: numpy restatement == the
    library's host table, bit for bit; it is a standard normal."""
    from paper_2305_04359_b200 import datagen
    from paper_2305_04359_b200._lib import check, lib
    want = np.empty(65536, np.float32)
    check(lib().gann_normal_table(want.ctypes.data))
    got = datagen.normal_table()
    assert (got == want).all()
    assert (got[::-1] == -got).all()  # symmetric
    assert abs(float(got.astype(np.float64).mean())) < 1e-9
    assert abs(float(got.astype(np.float64).std()) - 1.0) < 2e-3
    assert 4.3 < float(got.max()) < 4.35
    from math import erf, sqrt
    for zq in (-2.0, -1.0, 0.5, 1.5):  # empirical CDF of the 2^16 levels == Phi
        assert abs((got <= zq).mean() - 0.5 * (1 + erf(zq / sqrt(2)))) < 2e-5


def test_datagen_matches_config_distribution():
    """Noise ~ N(0, sigma^2) around U[0,255] centres (BASELINE configs 0/1),
    10% uniform rows for config 2."""
    from paper_2305_04359_b200 import datagen
    from paper_2305_04359_b200.datagen import K_CENTER, K_CLUSTER, mix64_2
    n, d, cl, sig = 4000, 128, 1000, 20.0
    x = datagen.gen_u8_numpy(n, d, cl, sig, 0.0, 1, 2).astype(np.float64)
    r = np.arange(n, dtype=np.uint64)[:, None]
    c = mix64_2(np.uint64(2) ^ K_CLUSTER, r) % np.uint64(cl)
    centre = (mix64_2(np.uint64(1) ^ K_CENTER, c * np.uint64(d) + np.arange(d, dtype=np.uint64)[None, :])
              >> np.uint64(56)).astype(np.float64)
    inner = (centre > 70) & (centre < 185)  # away from clipping
    noise = (x - centre)[inner]
    assert abs(noise.mean()) < 0.2 and abs(noise.std() - sig) < 0.6
    assert 0 <= centre.min() and centre.max() <= 255 and centre.std() > 70
    y = datagen.gen_u8_numpy(20000, 16, 5000, 12.0, 0.1, 1, 5)
    assert y.shape == (20000, 16)


def test_f32_datagen_config3_shape():
    """Config 3 (TTI-like): per-point norms log-normal(0, 0.3); queries from
    shifted centres are out of distribution (farther from their cluster)."""
    from paper_2305_04359_b200 import datagen
    cfg = datagen.CONFIGS["c3"].scaled(3000, 2000)
    x = datagen.host_base(cfg)
    q = datagen.host_queries(cfg)
    assert x.dtype == np.float32 and x.shape == (3000, 200) and q.shape == (2000, 200)
    ln = np.log(np.linalg.norm(x.astype(np.float64), axis=1))
    assert abs(ln.mean()) < 0.03 and abs(ln.std() - 0.3) < 0.03
    assert (datagen.gen_f32_numpy(100, 200, 2000, 0.5, 0.3, 0.0, 1, 2, row0=50) == x[50:150]).all()
    # the cosine to the unshifted centre is lower for the shifted (query) stream
    from paper_2305_04359_b200.datagen import K_CENTER, K_CLUSTER, _normal, mix64_2

    def cos_to_centre(rows, seed):
        r = np.arange(len(rows), dtype=np.uint64)[:, None]
        c = mix64_2(np.uint64(seed) ^ K_CLUSTER, r) % np.uint64(2000)
        cen = _normal(mix64_2(np.uint64(1) ^ K_CENTER, c * np.uint64(200) + np.arange(200, dtype=np.uint64)[None, :]))
        return (rows * cen).sum(1) / np.linalg.norm(rows, axis=1) / np.linalg.norm(cen, axis=1)

    assert cos_to_centre(q.astype(np.float64), cfg.query_seed).mean() < cos_to_centre(x.astype(np.float64)[:2000], cfg.base_seed).mean() - 0.02


def test_recall_tie_rule():
    """recall_k_at_n tie rule (reference src/eval.cpp:14-33, tests/test_eval.cpp:12-38)."""
    from paper_2305_04359_b200.evalutil import recall_at_k
    ti = np.array([[5, 6, 7, 8]], np.uint32)
    td = np.array([[1.0, 2.0, 2.0, 3.0]], np.float32)
    assert recall_at_k(ti, td, np.array([[5, 6]], np.uint32), 2)[0] == 1.0
    assert recall_at_k(ti, td, np.array([[5, 7]], np.uint32), 2)[0] == 1.0  # tie with the k-th distance
    assert recall_at_k(ti, td, np.array([[5, 8]], np.uint32), 2)[0] == 0.5
    assert recall_at_k(ti, td, np.array([[9, 8]], np.uint32), 2)[0] == 0.0


def test_recall_matches_reference(orc):
    from paper_2305_04359_b200.evalutil import recall_at_k
    rng = np.random.default_rng(3)
    ti = np.sort(rng.choice(1000, (50, 16)), axis=1).astype(np.uint32)
    td = np.sort(rng.integers(0, 5, (50, 16)).astype(np.float32), axis=1)
    res = rng.choice(1000, (50, 10)).astype(np.uint32)
    res[:, :4] = ti[:, :4]
    mine = recall_at_k(ti, td, res, 10)
    theirs = [orc.recall(ti[i], td[i], res[i], 10) for i in range(50)]
    assert np.allclose(mine, theirs)


def test_cpp_dropin_header_builds_and_links():
    """include/gann.hpp (the C++ mirror of graphann's API) compiles and links."""
    import subprocess
    subprocess.run(["make", "-s", "-C", str(ROOT / "tests" / "cpp")], check=True)
    exe = ROOT / "tests" / "cpp" / "_build" / "test_gann_cpp"
    assert exe.exists()
    out = subprocess.run(["nm", "-D", "--undefined-only", str(exe)], capture_output=True, text=True).stdout
    assert "gann_build" in out and "gann_search" in out


def test_bench_beam_rule():
    """bench.py's headline beam rule (both arms): smallest swept beam reaching
    the target, else past the sweep and bisected to a multiple of 32."""
    import argparse
    import bench
    args = argparse.Namespace(L=0, target_recall=0.95, no_extend=False)
    rec = lambda L: min(1.0, 0.8 + L / 5000.0)  # reaches 0.95 at L = 750
    curve = [{"L": L, "recall@10": rec(L)} for L in (10, 100, 200)]
    L, reached, ext = bench.choose_beam(args, curve, lambda L: (rec(L), {}))
    assert reached and L == 768 and rec(L) >= 0.95 and rec(L - 32) < 0.95
    assert [e["L"] for e in ext] == sorted(e["L"] for e in ext)
    L, reached, ext = bench.choose_beam(args, curve, lambda L: (rec(L), {}), max_beam=512)
    assert not reached and L == 512
    curve[1]["recall@10"] = 0.96
    assert bench.choose_beam(args, curve, None)[:2] == (100, True)
