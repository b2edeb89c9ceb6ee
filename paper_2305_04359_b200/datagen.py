"""Seeded synthetic inputs with the BASELINE configs' shapes and value distributions.

The paper measures on BIGANN / SSNPP / TTI (``PAPER.md:915-917``); none of
those datasets is available here, so the BASELINE configs are restated as
Gaussian mixtures (``BASELINE.json`` configs 0-4). Generation is a pure
function of (seeds, row, column): the device kernel (``csrc/misc.cu``,
``gann_generate_u8``) writes rows straight into HBM, and :func:`gen_u8_numpy`
restates it bit-for-bit on the host (tests pin the two together) so the CPU
reference arm can regenerate any prefix without a GPU.

Noise is Irwin-Hall(4) over 16-bit uniforms (unit variance): integer
arithmetic plus three IEEE f32 operations, identical on host and device.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
K_CENTER = np.uint64(0xC3A5C85C97CB3127)
K_CLUSTER = np.uint64(0x2545F4914F6CDD1D)
K_NOISE_ROW = np.uint64(0x9E3779B97F4A7C15)
K_UNIFORM = np.uint64(0xD6E8FEB86659FD93)
K_NORMAL = np.uint64(0xA0761D6478BD642F)


def mix64(x):
    """splitmix64 finaliser (reference include/graphann/core.hpp:47-53), vectorised."""
    with np.errstate(over="ignore"):
        x = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def mix64_2(a, b):
    return mix64(np.asarray(a, np.uint64) ^ mix64(b))


def gen_u8_numpy(n, d, clusters, sigma, noise_frac, center_seed, stream_seed, row0=0):
    """Host restatement of ``gen_u8_kernel`` (csrc/misc.cu)."""
    r = np.arange(row0, row0 + n, dtype=np.uint64)[:, None]
    j = np.arange(d, dtype=np.uint64)[None, :]
    el = r * np.uint64(d) + j
    thr = np.uint64(int(float(noise_frac) * 16777216.0))
    noise_row = (mix64_2(np.uint64(stream_seed) ^ K_NOISE_ROW, r) >> np.uint64(40)) < thr
    c = mix64_2(np.uint64(stream_seed) ^ K_CLUSTER, r) % np.uint64(clusters)
    center = (mix64_2(np.uint64(center_seed) ^ K_CENTER, c * np.uint64(d) + j) >> np.uint64(56)).astype(np.float32)
    h = mix64_2(np.uint64(stream_seed) ^ K_NORMAL, el)
    s = ((h & np.uint64(0xFFFF)) + ((h >> np.uint64(16)) & np.uint64(0xFFFF)) +
         ((h >> np.uint64(32)) & np.uint64(0xFFFF)) + ((h >> np.uint64(48)) & np.uint64(0xFFFF))).astype(np.int64)
    s = (s - 131070).astype(np.float32)
    inv_sd = np.float32(1.0) / np.float32(37837.2227)
    z = s * inv_sd
    x = center + np.float32(sigma) * z
    v = np.clip(np.rint(x), 0, 255).astype(np.uint8)
    uni = (mix64_2(np.uint64(stream_seed) ^ K_UNIFORM, el) >> np.uint64(56)).astype(np.uint8)
    return np.where(noise_row, uni, v)


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config as a synthetic workload."""
    name: str
    n: int
    d: int
    dtype: str
    metric: str
    clusters: int
    sigma: float
    noise_frac: float
    R: int
    L: int
    alpha: float
    batch_cap_frac: float  # 0 = uncapped prefix doubling
    n_queries: int = 10_000
    k: int = 10
    center_seed: int = 1
    base_seed: int = 2
    query_seed: int = 3

    @property
    def max_batch(self) -> int:
        return int(self.n * self.batch_cap_frac) if self.batch_cap_frac else 0

    def scaled(self, n: int, n_queries: int | None = None) -> "Config":
        from dataclasses import replace
        return replace(self, n=n, n_queries=self.n_queries if n_queries is None else n_queries)


CONFIGS = {
    # BASELINE.json configs[0]: 100k x 128 u8, 1000 clusters, sigma 20, batches capped at 2% of n
    "c0": Config("c0-100k-u8-d128", 100_000, 128, "u8", "l2", 1000, 20.0, 0.0, 64, 128, 1.2, 0.02),
    # configs[1]: the same generator at 10M (the 2% cap kept)
    "c1": Config("c1-10M-u8-d128", 10_000_000, 128, "u8", "l2", 1000, 20.0, 0.0, 64, 128, 1.2, 0.02),
    # configs[2]: 10M x 256 u8, 5000 clusters, sigma 12, 10% uniform noise points
    "c2": Config("c2-10M-u8-d256", 10_000_000, 256, "u8", "l2", 5000, 12.0, 0.10, 64, 128, 1.2, 0.02),
    # configs[4]: 1B x 128 u8 with 100k clusters (multi-GPU build; not runnable on one GPU)
    "c4": Config("c4-1B-u8-d128", 1_000_000_000, 128, "u8", "l2", 100_000, 20.0, 0.0, 64, 128, 1.2, 0.02),
}


def host_base(cfg: Config, n: int | None = None) -> np.ndarray:
    """Base points [0, n) of a config on the host (numpy restatement)."""
    n = cfg.n if n is None else n
    return gen_u8_numpy(n, cfg.d, cfg.clusters, cfg.sigma, cfg.noise_frac, cfg.center_seed, cfg.base_seed)


def host_queries(cfg: Config, nq: int | None = None) -> np.ndarray:
    nq = cfg.n_queries if nq is None else nq
    return gen_u8_numpy(nq, cfg.d, cfg.clusters, cfg.sigma, cfg.noise_frac, cfg.center_seed, cfg.query_seed)
