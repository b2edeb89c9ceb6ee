"""Recall scoring shared by bench.py and the tests (numpy, host side).

``recall_at_k`` restates graphann::recall_k_at_n (reference src/eval.cpp:14-33):
a result id is a hit if it is among the first k truth ids, or if it appears
later in the truth list at exactly the k-th truth distance (ties count).
"""
from __future__ import annotations

import numpy as np


def recall_at_k(truth_ids: np.ndarray, truth_dists: np.ndarray, result: np.ndarray, k: int) -> np.ndarray:
    """Per-query recall@k; truth arrays are (nq, depth >= k) sorted by (dist, id)."""
    truth_ids = np.asarray(truth_ids)
    truth_dists = np.asarray(truth_dists)
    result = np.asarray(result)
    nq, depth = truth_ids.shape
    if depth < k:
        raise ValueError("recall: ground truth depth below k")
    kth = truth_dists[:, k - 1:k]
    allowed = np.zeros_like(truth_ids, dtype=bool)
    allowed[:, :k] = True
    if depth > k:
        allowed[:, k:] = truth_dists[:, k:] == kth
    hits = np.zeros(nq, np.int64)
    for j in range(result.shape[1]):
        r = result[:, j:j + 1]
        hits += ((truth_ids == r) & allowed).any(axis=1) & (r[:, 0] != 0xFFFFFFFF)
    return np.minimum(hits, k) / k


# ---- batched eval harness ----------------------------------
# graphann's run_sweep / pareto_frontier / write_csv (include/graphann/eval.hpp,
# src/eval.cpp:104-254), restated for a batched GPU search: a sweep point is one
# call over all queries instead of a thread pool over per-query calls.
import sys
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence


@dataclass
class SweepConfig:
    beams: List[int]
    ks: List[int]
    epsilons: List[float]
    repetitions: int = 1


@dataclass
class EvalMeta:
    algorithm: str = ""
    dataset: str = ""
    n: int = 0
    build_seconds: float = 0.0
    threads: int = 1            # the CSV's "# threads=" line: GPUs for the batched search


@dataclass
class EvalRow:
    beam: int = 0
    k: int = 0
    epsilon: float = 0.0
    recall: float = 0.0
    qps: float = 0.0
    latency_ms: float = 0.0
    dist_comps: float = 0.0


@dataclass
class EvalReport:
    meta: EvalMeta
    rows: List[EvalRow] = field(default_factory=list)


def _validate_sweep(sweep: SweepConfig) -> None:
    # src/eval.cpp:104-113
    if not sweep.beams or not sweep.epsilons or not sweep.ks:
        raise ValueError("sweep: parameter lists must be nonempty")
    for e in sweep.epsilons:
        if e < 0.0 or e > 0.25:
            raise ValueError("sweep: epsilon outside [0, 0.25]")
    if sweep.repetitions == 0:
        raise ValueError("sweep: repetitions must be positive")


def _row_key(r: EvalRow):
    # sort_rows, src/eval.cpp:115-123: recall, qps, beam, k, epsilon ascending
    return (r.recall, r.qps, r.beam, r.k, r.epsilon)


# search(beam, k, eps) -> (ids (nq, k), dist_comps (nq,)) for ALL queries in one call
BatchSearch = Callable[[int, int, float], tuple]


def run_sweep(search: BatchSearch, truth_ids: np.ndarray, truth_dists: np.ndarray, sweep: SweepConfig,
              meta: EvalMeta, clock: Callable[[], float] = None) -> EvalReport:
    """graphann::run_sweep (src/eval.cpp:127-168) over a batched search.
    One row per (beam, k, eps) with k <= beam (others are skipped with a note on
    stderr), sorted by recall ascending. qps is the best repetition's
    nq / wall time of the batched call; latency_ms is the mean wall time of a
    call (every query of a batch completes with the batch); dist_comps is the
    mean per query over every repetition; recall uses the first repetition's ids."""
    import time
    clock = clock or time.perf_counter
    _validate_sweep(sweep)
    truth_ids = np.asarray(truth_ids)
    nq, depth = truth_ids.shape
    for k in sweep.ks:
        if k == 0 or k > depth:
            raise ValueError("sweep: ground truth depth below k")
    report = EvalReport(meta=meta)
    for beam in sweep.beams:
        for k in sweep.ks:
            if k > beam:
                print(f"note: skipping sweep point beam={beam} k={k} (k exceeds beam)", file=sys.stderr)
                continue
            for eps in sweep.epsilons:
                best, secs, dcs, first = float("inf"), [], [], None
                for rep in range(sweep.repetitions):
                    t0 = clock()
                    ids, dc = search(beam, k, eps)
                    dt = clock() - t0
                    best = min(best, dt)
                    secs.append(dt)
                    dcs.append(np.asarray(dc, np.float64).mean() if nq else 0.0)
                    if first is None:
                        first = np.asarray(ids)
                rec = float(recall_at_k(truth_ids, truth_dists, first, k).mean()) if nq else 0.0
                report.rows.append(EvalRow(beam, k, float(np.float32(eps)), rec, nq / best if best > 0 else 0.0,
                                           1e3 * float(np.mean(secs)), float(np.mean(dcs))))
    report.rows.sort(key=_row_key)
    return report


def pareto_frontier(rows: Sequence[EvalRow]) -> List[EvalRow]:
    """graphann::pareto_frontier (src/eval.cpp:205-225): rows not dominated in
    (recall, qps), recall ascending; duplicates collapse."""
    srt = sorted(rows, key=lambda r: (-r.recall, -r.qps, r.beam, r.k, r.epsilon))
    keep, best = [], -1.0
    for r in srt:
        if r.qps > best:
            keep.append(r)
            best = r.qps
    keep.reverse()
    return keep


def write_csv(report: EvalReport, out) -> None:
    """graphann::write_csv (src/eval.cpp:236-245): a "# threads=N" line, the
    header, one line per row; numbers as printf %.6g."""
    f = lambda v: "%.6g" % v  # noqa: E731
    m = report.meta
    out.write(f"# threads={m.threads}\n")
    out.write("algorithm,dataset,n,build_seconds,beam,k,epsilon,recall,qps,latency_ms,dist_comps\n")
    for r in report.rows:
        out.write(f"{m.algorithm},{m.dataset},{m.n},{f(m.build_seconds)},{r.beam},{r.k},{f(r.epsilon)},"
                  f"{f(r.recall)},{f(r.qps)},{f(r.latency_ms)},{f(r.dist_comps)}\n")
