"""Seeded small inputs for the parity tests (numpy only)."""
import numpy as np


def mixture(seed, n, d, clusters=8, sigma=20.0, dtype=np.uint8, nq=0):
    """Gaussian-mixture points (and optionally held-out queries) of a dtype."""
    rng = np.random.default_rng(seed)
    if dtype == np.float32:
        centers = rng.normal(0, 1, (clusters, d))
        pts = centers[rng.integers(0, clusters, n + nq)] + rng.normal(0, 1, (n + nq, d))
        pts = pts.astype(np.float32)
    elif dtype == np.int8:
        centers = rng.integers(-128, 128, (clusters, d))
        pts = np.clip(np.rint(centers[rng.integers(0, clusters, n + nq)] + rng.normal(0, sigma, (n + nq, d))),
                      -128, 127).astype(np.int8)
    else:
        centers = rng.integers(0, 256, (clusters, d))
        pts = np.clip(np.rint(centers[rng.integers(0, clusters, n + nq)] + rng.normal(0, sigma, (n + nq, d))),
                      0, 255).astype(np.uint8)
    return (pts[:n], pts[n:]) if nq else pts


def degrees(adj):
    return (np.asarray(adj) != 0xFFFFFFFF).sum(axis=1)
