"""Batched eval harness: run_sweep / pareto_frontier /
write_csv of evalutil against graphann's own (src/eval.cpp:104-254) — CPU only."""
import io

import numpy as np
import pytest

from paper_2305_04359_b200 import evalutil as E


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Oracle, available
    if not available("ref"):
        pytest.skip("needs oracle/_ref")
    return Oracle("ref")


def random_rows(seed, n):
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        rec = float(rng.choice([0.5, 0.75, 0.9, 0.95, 0.99, 1.0])) if i % 3 == 0 else float(rng.random())
        qps = float(rng.choice([1e3, 2.5e4])) if i % 4 == 0 else float(10 ** rng.uniform(2, 8))
        rows.append(E.EvalRow(int(rng.integers(1, 300)), int(rng.integers(1, 20)),
                              float(np.float32(rng.choice([0.0, 0.1, 0.25]))), rec, qps,
                              float(10 ** rng.uniform(-4, 2)), float(rng.uniform(10, 1e5))))
    rows += rows[:3]  # exact duplicates collapse
    return rows


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_pareto_frontier_matches_reference(ref, seed):
    rows = random_rows(seed, 60)
    ours = [(r.beam, r.k, r.epsilon, r.recall, r.qps) for r in E.pareto_frontier(rows)]
    assert ours == ref.pareto(rows)


def test_write_csv_byte_identical(ref, tmp_path):
    rows = random_rows(4, 25)
    meta = E.EvalMeta("diskann", "c1-10M-u8-d128", 10_000_000, 4.0912345678, 1)
    buf = io.StringIO()
    E.write_csv(E.EvalReport(meta, rows), buf)
    ref.write_csv(meta, rows, tmp_path / "ref.csv")
    assert buf.getvalue() == (tmp_path / "ref.csv").read_text()


def fake_search(truth):
    """A batched search returning the truth ids shifted by `beam % 3` columns."""
    def search(beam, k, eps):
        sh = beam % 3
        ids = np.roll(truth[:, :k], -sh, axis=1).copy()
        if sh:
            ids[:, k - sh:] = 0xFFFFFFFF
        return ids, np.full(len(truth), beam * 10.0 + k)
    return search


def test_run_sweep_rows_sorted_skips_and_validates(capsys):
    rng = np.random.default_rng(5)
    nq, depth = 50, 20
    truth = np.stack([rng.permutation(1000)[:depth] for _ in range(nq)]).astype(np.uint32)
    tdist = np.sort(rng.random((nq, depth)).astype(np.float32), axis=1)
    sweep = E.SweepConfig(beams=[4, 10, 12], ks=[5, 10], epsilons=[0.0, 0.1], repetitions=2)
    rep = E.run_sweep(fake_search(truth), truth, tdist, sweep, E.EvalMeta("x", "y", 1000))
    assert "skipping sweep point beam=4 k=5" in capsys.readouterr().err
    assert len(rep.rows) == 2 * 2 * 2  # beam 4 has no k <= 4: both skipped
    keys = [(r.recall, r.qps, r.beam, r.k, r.epsilon) for r in rep.rows]
    assert keys == sorted(keys)
    for r in rep.rows:  # recall of the shifted truth: (k - shift) / k
        assert r.recall == pytest.approx((r.k - r.beam % 3) / r.k)
        assert r.dist_comps == r.beam * 10.0 + r.k and r.qps > 0 and r.latency_ms >= 0
    with pytest.raises(ValueError):
        E.run_sweep(fake_search(truth), truth, tdist, E.SweepConfig([], [10], [0.0]), E.EvalMeta())
    with pytest.raises(ValueError):
        E.run_sweep(fake_search(truth), truth, tdist, E.SweepConfig([10], [10], [0.3]), E.EvalMeta())
    with pytest.raises(ValueError):
        E.run_sweep(fake_search(truth), truth, tdist, E.SweepConfig([10], [10], [0.0], 0), E.EvalMeta())
    with pytest.raises(ValueError):
        E.run_sweep(fake_search(truth), truth, tdist, E.SweepConfig([30], [25], [0.0]), E.EvalMeta())
