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
