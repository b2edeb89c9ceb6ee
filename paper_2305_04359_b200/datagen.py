"""Seeded synthetic inputs with the BASELINE configs' shapes and value distributions.

The paper measures on BIGANN / SSNPP / TTI (``PAPER.md:915-917``); none of
those datasets is available here, so the BASELINE configs are restated as
Gaussian mixtures (``BASELINE.json`` configs 0-4). Generation is a pure
function of (seeds, row, column): the device kernel (``csrc/misc.cu``,
``gann_generate_u8``) writes rows straight into HBM, and :func:`gen_u8_numpy`
restates it bit-for-bit on the host (tests pin the two together) so the CPU
reference arm can regenerate any prefix without a GPU.

Noise is Gaussian: a deviate is the normal quantile of a 16-bit uniform,
``z = Phi^-1((u + 1/2) / 2^16)``, read from a 65,536-entry table on a 2^-16
grid (:func:`normal_table`; the library's ``gann_normal_table`` computes the
same table and a CPU test pins the two), so host and device agree exactly.
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
K_SHIFT = np.uint64(0x8CB92BA72F3D8DD7)
K_NORM = np.uint64(0x3C6EF372FE94F82B)


def mix64(x):
    """splitmix64 finaliser (reference include/graphann/core.hpp:47-53), vectorised."""
    with np.errstate(over="ignore"):
        x = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def mix64_2(a, b):
    return mix64(np.asarray(a, np.uint64) ^ mix64(b))


_ACKLAM_A = (-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
             1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00)
_ACKLAM_B = (-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
             6.680131188771972e+01, -1.328068155288572e+01)
_ACKLAM_C = (-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
             -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00)
_ACKLAM_D = (7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00, 3.754408661907416e+00)


def _norm_ppf(p):
    """Phi^-1(p): Acklam's rational approximation + one Halley step on erfc
    (restates ``norm_ppf`` in csrc/misc.cu with the same libm calls)."""
    import math
    a, b, c, d = _ACKLAM_A, _ACKLAM_B, _ACKLAM_C, _ACKLAM_D
    plow = 0.02425
    if p < plow:
        q = math.sqrt(-2.0 * math.log(p))
        x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) / \
            ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0)
    elif p <= 1.0 - plow:
        q = p - 0.5
        r = q * q
        x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q / \
            (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0)
    else:
        q = math.sqrt(-2.0 * math.log(1.0 - p))
        x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) / \
            ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0)
    e = 0.5 * math.erfc(-x / math.sqrt(2.0)) - p
    u = e * math.sqrt(2.0 * 3.14159265358979323846) * math.exp(x * x / 2.0)
    return x - u / (1.0 + x * u / 2.0)


_NTAB = None


def normal_table() -> np.ndarray:
    """float32[65536]: table[u] = Phi^-1((u + 1/2) / 2^16) rounded to a 2^-16 grid."""
    global _NTAB
    if _NTAB is None:
        t = np.array([round(_norm_ppf((u + 0.5) / 65536.0) * 65536.0) / 65536.0 for u in range(65536)],
                     dtype=np.float64)
        _NTAB = t.astype(np.float32)
    return _NTAB


def gen_u8_numpy(n, d, clusters, sigma, noise_frac, center_seed, stream_seed, row0=0):
    """Host restatement of ``gen_u8_kernel`` (csrc/misc.cu)."""
    r = np.arange(row0, row0 + n, dtype=np.uint64)[:, None]
    j = np.arange(d, dtype=np.uint64)[None, :]
    el = r * np.uint64(d) + j
    thr = np.uint64(int(float(noise_frac) * 16777216.0))
    noise_row = (mix64_2(np.uint64(stream_seed) ^ K_NOISE_ROW, r) >> np.uint64(40)) < thr
    c = mix64_2(np.uint64(stream_seed) ^ K_CLUSTER, r) % np.uint64(clusters)
    center = (mix64_2(np.uint64(center_seed) ^ K_CENTER, c * np.uint64(d) + j) >> np.uint64(56)).astype(np.float32)
    z = normal_table()[(mix64_2(np.uint64(stream_seed) ^ K_NORMAL, el) & np.uint64(0xFFFF)).astype(np.int64)]
    x = center + np.float32(sigma) * z
    v = np.clip(np.rint(x), 0, 255).astype(np.uint8)
    uni = (mix64_2(np.uint64(stream_seed) ^ K_UNIFORM, el) >> np.uint64(56)).astype(np.uint8)
    return np.where(noise_row, uni, v)


def _normal(h):
    """The N(0, 1) deviate of hash h: normal_table()[h & 0xFFFF], as float64."""
    return normal_table()[(h & np.uint64(0xFFFF)).astype(np.int64)].astype(np.float64)


def gen_f32_numpy(n, d, clusters, sigma, norm_sigma, shift, center_seed, stream_seed, row0=0):
    """Host restatement of ``gen_f32_kernel`` (csrc/misc.cu): double arithmetic,
    one rounding to f32 (the device's warp-order sum of squares may differ in
    the last double bit, so compare with a ~1e-6 relative tolerance)."""
    r = np.arange(row0, row0 + n, dtype=np.uint64)[:, None]
    j = np.arange(d, dtype=np.uint64)[None, :]
    c = mix64_2(np.uint64(stream_seed) ^ K_CLUSTER, r) % np.uint64(clusters)
    v = _normal(mix64_2(np.uint64(center_seed) ^ K_CENTER, c * np.uint64(d) + j))
    if shift > 0:
        v = v + float(np.float32(shift)) * _normal(mix64_2(np.uint64(center_seed) ^ K_SHIFT, c * np.uint64(d) + j))
    v = v + float(np.float32(sigma)) * _normal(mix64_2(np.uint64(stream_seed) ^ K_NORMAL, r * np.uint64(d) + j))
    g = _normal(mix64_2(np.uint64(stream_seed) ^ K_NORM, r))
    scale = np.exp(float(np.float32(norm_sigma)) * g) / np.sqrt((v * v).sum(axis=1, keepdims=True))
    return (v * scale).astype(np.float32)


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
    norm_sigma: float = 0.0   # f32 configs: log-normal sigma of the per-point norms
    query_shift: float = 0.0  # f32 configs: queries from centres shifted by N(0, shift^2)

    @property
    def np_dtype(self):
        return {"u8": np.uint8, "i8": np.int8, "f32": np.float32}[self.dtype]

    @property
    def elem_bytes(self) -> int:
        return np.dtype(self.np_dtype).itemsize

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
    # configs[3]: 10M x 200 f32, negative inner product, 2000-component mixture,
    # log-normal(0, 0.3) per-point norms, out-of-distribution queries (centres
    # shifted by N(0, 0.5)), alpha 1.0 (TTI-like)
    "c3": Config("c3-10M-f32-d200-ip", 10_000_000, 200, "f32", "ip", 2000, 0.5, 0.0, 64, 128, 1.0, 0.02,
                 norm_sigma=0.3, query_shift=0.5),
    # configs[4]: 1B x 128 u8 with 100k clusters (multi-GPU build; not runnable on one GPU)
    "c4": Config("c4-1B-u8-d128", 1_000_000_000, 128, "u8", "l2", 100_000, 20.0, 0.0, 64, 128, 1.2, 0.02),
}


def host_base(cfg: Config, n: int | None = None) -> np.ndarray:
    """Base points [0, n) of a config on the host (numpy restatement)."""
    n = cfg.n if n is None else n
    if cfg.dtype == "f32":
        return gen_f32_numpy(n, cfg.d, cfg.clusters, cfg.sigma, cfg.norm_sigma, 0.0, cfg.center_seed, cfg.base_seed)
    return gen_u8_numpy(n, cfg.d, cfg.clusters, cfg.sigma, cfg.noise_frac, cfg.center_seed, cfg.base_seed)


def _u8_rows_fast(out, row0, n, d, clusters, sigma, noise_frac, center_seed, stream_seed, centers):
    """gen_u8_numpy for rows [row0, row0+n) into out[row0:row0+n], with the
    cluster centres precomputed (the same values, fewer hashes)."""
    r = np.arange(row0, row0 + n, dtype=np.uint64)[:, None]
    c = (mix64_2(np.uint64(stream_seed) ^ K_CLUSTER, r) % np.uint64(clusters)).astype(np.int64)
    el = r * np.uint64(d) + np.arange(d, dtype=np.uint64)[None, :]
    z = normal_table()[(mix64_2(np.uint64(stream_seed) ^ K_NORMAL, el) & np.uint64(0xFFFF)).astype(np.int64)]
    x = centers[c[:, 0]] + np.float32(sigma) * z
    v = np.clip(np.rint(x), 0, 255).astype(np.uint8)
    if noise_frac > 0:
        thr = np.uint64(int(float(noise_frac) * 16777216.0))
        noise_row = (mix64_2(np.uint64(stream_seed) ^ K_NOISE_ROW, r) >> np.uint64(40)) < thr
        uni = (mix64_2(np.uint64(stream_seed) ^ K_UNIFORM, el) >> np.uint64(56)).astype(np.uint8)
        v = np.where(noise_row, uni, v)
    out[row0:row0 + n] = v


def host_base_parallel(cfg: Config, n: int | None = None, threads: int | None = None,
                       chunk: int = 65536) -> np.ndarray:
    """host_base for the u8 configs at full size: row chunks on a thread pool
    (numpy releases the GIL), cluster centres computed once. Bit-identical to
    gen_u8_numpy (tests pin it) and to the device generator."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    n = cfg.n if n is None else n
    if cfg.dtype == "f32":
        return host_base(cfg, n)
    d = cfg.d
    cj = np.arange(d, dtype=np.uint64)[None, :]
    cc = np.arange(cfg.clusters, dtype=np.uint64)[:, None]
    centers = (mix64_2(np.uint64(cfg.center_seed) ^ K_CENTER, cc * np.uint64(d) + cj) >> np.uint64(56)).astype(np.float32)
    out = np.empty((n, d), np.uint8)
    starts = range(0, n, chunk)
    with ThreadPoolExecutor(threads or os.cpu_count() or 1) as ex:
        list(ex.map(lambda r0: _u8_rows_fast(out, r0, min(chunk, n - r0), d, cfg.clusters, cfg.sigma, cfg.noise_frac,
                                             cfg.center_seed, cfg.base_seed, centers), starts))
    return out


def host_queries(cfg: Config, nq: int | None = None) -> np.ndarray:
    nq = cfg.n_queries if nq is None else nq
    if cfg.dtype == "f32":
        return gen_f32_numpy(nq, cfg.d, cfg.clusters, cfg.sigma, cfg.norm_sigma, cfg.query_shift, cfg.center_seed,
                             cfg.query_seed)
    return gen_u8_numpy(nq, cfg.d, cfg.clusters, cfg.sigma, cfg.noise_frac, cfg.center_seed, cfg.query_seed)


def generate_device(lib, cfg: Config, ptr: int, n: int, queries: bool, row0: int = 0, device: int = 0) -> int:
    """Rows [row0, row0+n) of a config's base (or query) stream straight into
    device memory at ptr (gann_generate_u8 / gann_generate_f32). Returns the C
    status code."""
    seed = cfg.query_seed if queries else cfg.base_seed
    if cfg.dtype == "f32":
        return lib.gann_generate_f32(ptr, n, cfg.d, cfg.clusters, cfg.sigma, cfg.norm_sigma,
                                     cfg.query_shift if queries else 0.0, cfg.center_seed, seed, row0, device)
    return lib.gann_generate_u8(ptr, n, cfg.d, cfg.clusters, cfg.sigma, cfg.noise_frac, cfg.center_seed, seed, row0,
                                device)
