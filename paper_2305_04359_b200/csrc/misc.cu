// misc.cu — start vertex, synthetic data generator, brute-force ground truth.
#include <algorithm>
#include <cub/device/device_radix_sort.cuh>
#include <cmath>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace gann {

namespace {

template <int E>
__device__ __forceinline__ float elem_at(const uint8_t* row, uint32_t j) {
  if (E == kU8) return static_cast<float>(row[j]);
  if (E == kI8) return static_cast<float>(reinterpret_cast<const int8_t*>(row)[j]);
  return reinterpret_cast<const float*>(row)[j];
}

// Column sums in double — builder_common.cpp:65-74. Exact for integer kinds
// whatever the summation order.
template <int E>
__global__ void colsum_kernel(const uint8_t* data, uint64_t stride, uint64_t n, uint32_t d,
                              double* colsum) {
  constexpr uint32_t kRows = 512;
  const uint64_t r0 = uint64_t(blockIdx.x) * kRows;
  const uint64_t r1 = min(n, r0 + kRows);
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) {
    double acc = 0.0;
    for (uint64_t r = r0; r < r1; r++) acc += static_cast<double>(elem_at<E>(data + r * stride, j));
    atomicAdd(colsum + j, acc);
  }
}

__global__ void centroid_kernel(const double* colsum, uint64_t n, uint32_t d, float* c) {
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x)
    c[j] = __double2float_rn(__ddiv_rn(colsum[j], static_cast<double>(n)));  // :76-80
}

// dist_to_centroid — builder_common.cpp:24-38: sequential float, no FMA.
template <int E, int M>
__global__ void start_dist_kernel(const uint8_t* data, uint64_t stride, uint64_t n, uint32_t d,
                                  const float* centroid, unsigned long long* best) {
  extern __shared__ float cs[];
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) cs[j] = centroid[j];
  __syncthreads();
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint64_t key = kMaxKey;
  if (i < n) {
    const uint8_t* row = data + i * stride;
    float acc = 0.0f;
    for (uint32_t j = 0; j < d; j++) {
      const float x = elem_at<E>(row, j);
      if (M == kL2) {
        const float diff = __fsub_rn(x, cs[j]);
        acc = __fadd_rn(acc, __fmul_rn(diff, diff));
      } else {
        acc = __fadd_rn(acc, __fmul_rn(x, cs[j]));
      }
    }
    key = make_key(M == kL2 ? acc : -acc, static_cast<uint32_t>(i));
  }
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t other = __shfl_xor_sync(0xFFFFFFFFu, key, o);
    key = other < key ? other : key;
  }
  if ((threadIdx.x & 31) == 0 && key != kMaxKey) atomicMin(best, static_cast<unsigned long long>(key));
}

// ---- synthetic data ---------------------------------------------------------
// A pure function of (seeds, row, column), restated bit-for-bit in numpy by
// paper_2305_04359_b200/datagen.py. A standard normal deviate is the Gaussian
// quantile of a 16-bit uniform, z = Phi^-1((u + 1/2) / 2^16), looked up in a
// 2^16-entry table (normal_table below: an exact Gaussian up to the 16-bit
// discretisation, tails to +-4.32 sigma) that host and device share, so the
// rest is IEEE f32 (u8 rows) or double (f32 rows) arithmetic on both sides.
constexpr uint64_t kKCenter = 0xC3A5C85C97CB3127ull;
constexpr uint64_t kKCluster = 0x2545F4914F6CDD1Dull;
constexpr uint64_t kKNoiseRow = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kKUniform = 0xD6E8FEB86659FD93ull;
constexpr uint64_t kKNormal = 0xA0761D6478BD642Full;

__global__ void gen_u8_kernel(uint8_t* out, uint64_t out_stride, uint64_t n, uint32_t d,
                              uint32_t clusters, float sigma, uint32_t noise_thr,
                              uint64_t cseed, uint64_t sseed, uint64_t row0, const float* __restrict__ ntab) {
  const uint64_t total = n * d;
  const uint64_t step = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += step) {
    const uint64_t i = idx / d;
    const uint32_t j = static_cast<uint32_t>(idx - i * d);
    const uint64_t r = row0 + i;
    const uint64_t el = r * d + j;
    uint32_t v;
    if ((mix64(sseed ^ kKNoiseRow, r) >> 40) < noise_thr) {
      v = static_cast<uint32_t>(mix64(sseed ^ kKUniform, el) >> 56);
    } else {
      const uint64_t c = mix64(sseed ^ kKCluster, r) % clusters;
      const uint32_t center = static_cast<uint32_t>(mix64(cseed ^ kKCenter, c * d + j) >> 56);
      const float z = __ldg(ntab + (mix64(sseed ^ kKNormal, el) & 0xFFFF));
      const float x = __fadd_rn(static_cast<float>(center), __fmul_rn(sigma, z));
      const float rx = rintf(x);
      v = rx < 0.0f ? 0u : (rx > 255.0f ? 255u : static_cast<uint32_t>(rx));
    }
    out[i * out_stride + j] = static_cast<uint8_t>(v);
  }
}

// f32 mixture rows (config 3): one warp per row. Normals come from the same
// quantile table; the rest is double arithmetic, one rounding to f32 at the
// end (datagen.gen_f32_numpy restates it).
constexpr uint64_t kKShift = 0x8CB92BA72F3D8DD7ull;
constexpr uint64_t kKNorm = 0x3C6EF372FE94F82Bull;

__global__ void gen_f32_kernel(float* out, uint64_t n, uint32_t d, uint32_t clusters, double sigma,
                               double norm_sigma, double shift, uint64_t cseed, uint64_t sseed, uint64_t row0,
                               const float* __restrict__ ntab) {
  auto ih_normal = [&](uint64_t h) { return static_cast<double>(__ldg(ntab + (h & 0xFFFF))); };
  const int lane = threadIdx.x & 31;
  const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const uint64_t r = row0 + i;
    const uint64_t c = mix64(sseed ^ kKCluster, r) % clusters;
    double ss = 0.0;
    for (uint32_t j = lane; j < d; j += 32) {
      double v = ih_normal(mix64(cseed ^ kKCenter, c * d + j));
      if (shift > 0.0) v += shift * ih_normal(mix64(cseed ^ kKShift, c * d + j));
      v += sigma * ih_normal(mix64(sseed ^ kKNormal, r * d + j));
      ss += v * v;
    }
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xFFFFFFFFu, ss, o);
    const double scale = exp(norm_sigma * ih_normal(mix64(sseed ^ kKNorm, r))) / sqrt(ss);
    for (uint32_t j = lane; j < d; j += 32) {
      double v = ih_normal(mix64(cseed ^ kKCenter, c * d + j));
      if (shift > 0.0) v += shift * ih_normal(mix64(cseed ^ kKShift, c * d + j));
      v += sigma * ih_normal(mix64(sseed ^ kKNormal, r * d + j));
      out[i * d + j] = static_cast<float>(v * scale);
    }
  }
}

// ---- brute-force ground truth ---------------------------------------------
// compute_groundtruth (src/dataset.cpp:172-217): exact top-k by (dist, id).
// One thread per query (its row in registers), a shared-memory tile of points
// broadcast to the block; the point range is split across blockIdx.y and the
// per-split top-16 lists are merged by gt_merge_kernel.
constexpr int kGtMaxK = 64;  // the largest k (gann_groundtruth)
constexpr int kGtThreads = 128;
constexpr int kGtTile = 128;

template <int E, int M, int NCH, int K>
__global__ void __launch_bounds__(kGtThreads)
    gt_kernel(const uint8_t* data, uint64_t stride, uint64_t n, const uint8_t* queries,
              uint32_t nq, uint32_t nch, uint32_t splits, unsigned long long* partial) {
  constexpr int kGtK = K;
  using Op = DistOp<E, M>;
  extern __shared__ __align__(16) uint4 tile[];
  const uint32_t q = blockIdx.x * kGtThreads + threadIdx.x;
  const uint64_t lo = n * blockIdx.y / splits, hi = n * (blockIdx.y + 1) / splits;
  uint4 qr[NCH];
#pragma unroll
  for (int c = 0; c < NCH; c++)
    qr[c] = (q < nq && c < static_cast<int>(nch))
                ? __ldg(reinterpret_cast<const uint4*>(queries + uint64_t(q) * stride) + c)
                : make_uint4(0, 0, 0, 0);
  uint64_t top[kGtK];
#pragma unroll
  for (int i = 0; i < kGtK; i++) top[i] = kMaxKey;
  for (uint64_t p0 = lo; p0 < hi; p0 += kGtTile) {
    const uint32_t cnt = static_cast<uint32_t>((hi - p0) < kGtTile ? (hi - p0) : uint64_t(kGtTile));
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < cnt * nch; t += kGtThreads) {
      const uint32_t pp = t / nch, c = t - pp * nch;
      tile[pp * NCH + c] = __ldg(reinterpret_cast<const uint4*>(data + (p0 + pp) * stride) + c);
    }
    __syncthreads();
    for (uint32_t pp = 0; pp < cnt; pp++) {
      typename Op::acc_t acc = Op::zero();
#pragma unroll
      for (int c = 0; c < NCH; c++)
        if (c < static_cast<int>(nch)) acc = Op::chunk(qr[c], tile[pp * NCH + c], acc);
      const uint64_t key = make_key(Op::finish(acc), static_cast<uint32_t>(p0 + pp));
      if (key < top[kGtK - 1]) {
        top[kGtK - 1] = key;
#pragma unroll
        for (int i = kGtK - 1; i > 0; i--) {
          if (top[i] < top[i - 1]) {
            const uint64_t t = top[i];
            top[i] = top[i - 1];
            top[i - 1] = t;
          }
        }
      }
    }
  }
  if (q < nq) {
    unsigned long long* out = partial + (uint64_t(q) * splits + blockIdx.y) * kGtK;
#pragma unroll
    for (int i = 0; i < kGtK; i++) out[i] = top[i];
  }
}

// Rows above 256 bytes: the block's 128 query rows live in shared memory
// (thread = query, as above), the point tile beside them.
template <int E, int M, int K>
__global__ void __launch_bounds__(kGtThreads)
    gt_wide_kernel(const uint8_t* data, uint64_t stride, uint64_t n, const uint8_t* queries, uint32_t nq,
                   uint32_t nch, uint32_t splits, uint32_t tile_pts, unsigned long long* partial) {
  using Op = DistOp<E, M>;
  extern __shared__ __align__(16) uint4 sm[];
  uint4* qs = sm;                           // kGtThreads rows of nch chunks
  uint4* tile = sm + size_t(kGtThreads) * nch;  // tile_pts rows
  const uint32_t q = blockIdx.x * kGtThreads + threadIdx.x;
  const uint64_t lo = n * blockIdx.y / splits, hi = n * (blockIdx.y + 1) / splits;
  for (uint32_t t = threadIdx.x; t < kGtThreads * nch; t += kGtThreads) {
    const uint32_t qq = blockIdx.x * kGtThreads + t / nch, c = t % nch;
    qs[t] = qq < nq ? __ldg(reinterpret_cast<const uint4*>(queries + uint64_t(qq) * stride) + c) : make_uint4(0, 0, 0, 0);
  }
  uint64_t top[K];
  for (int i = 0; i < K; i++) top[i] = kMaxKey;
  const uint4* my = qs + size_t(threadIdx.x) * nch;
  for (uint64_t p0 = lo; p0 < hi; p0 += tile_pts) {
    const uint32_t cnt = static_cast<uint32_t>((hi - p0) < tile_pts ? (hi - p0) : uint64_t(tile_pts));
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < cnt * nch; t += kGtThreads) {
      const uint32_t pp = t / nch, c = t - pp * nch;
      tile[t] = __ldg(reinterpret_cast<const uint4*>(data + (p0 + pp) * stride) + c);
    }
    __syncthreads();
    for (uint32_t pp = 0; pp < cnt; pp++) {
      typename Op::acc_t acc = Op::zero();
      for (uint32_t c = 0; c < nch; c++) acc = Op::chunk(my[c], tile[pp * nch + c], acc);
      const uint64_t key = make_key(Op::finish(acc), static_cast<uint32_t>(p0 + pp));
      if (key < top[K - 1]) {
        int i = K - 1;
        for (; i > 0 && top[i - 1] > key; i--) top[i] = top[i - 1];
        top[i] = key;
      }
    }
  }
  if (q < nq) {
    unsigned long long* out = partial + (uint64_t(q) * splits + blockIdx.y) * K;
    for (int i = 0; i < K; i++) out[i] = top[i];
  }
}

template <int K>
__global__ void gt_merge_kernel(const unsigned long long* partial, uint32_t nq, uint32_t splits,
                                uint32_t k, uint32_t* ids, float* dists) {
  constexpr int kGtK = K;
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  uint64_t top[kGtK];
#pragma unroll
  for (int i = 0; i < kGtK; i++) top[i] = kMaxKey;
  const unsigned long long* in = partial + uint64_t(q) * splits * kGtK;
  for (uint32_t t = 0; t < splits * kGtK; t++) {
    const uint64_t key = in[t];
    if (key < top[kGtK - 1]) {
      top[kGtK - 1] = key;
#pragma unroll
      for (int i = kGtK - 1; i > 0; i--) {
        if (top[i] < top[i - 1]) {
          const uint64_t x = top[i];
          top[i] = top[i - 1];
          top[i - 1] = x;
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kGtK; i++) {
    if (static_cast<uint32_t>(i) < k) {
      ids[uint64_t(q) * k + i] = top[i] == kMaxKey ? kNone : key_id(top[i]);
      dists[uint64_t(q) * k + i] = top[i] == kMaxKey ? __int_as_float(0x7f800000) : key_dist(top[i]);
    }
  }
}

template <int E, int M, int NCH, int K>
cudaError_t gt_launch(const uint8_t* data, uint64_t stride, uint64_t n, const uint8_t* queries,
                      uint32_t nq, uint32_t nch, uint32_t splits, unsigned long long* partial,
                      cudaStream_t s) {
  const size_t smem = size_t(kGtTile) * NCH * 16;
  auto k = gt_kernel<E, M, NCH, K>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  dim3 grid((nq + kGtThreads - 1) / kGtThreads, splits);
  k<<<grid, kGtThreads, smem, s>>>(data, stride, n, queries, nq, nch, splits, partial);
  return cudaGetLastError();
}

template <int E, int M, int K>
cudaError_t gt_dispatch_k(const uint8_t* data, uint64_t stride, uint64_t n, const uint8_t* queries,
                          uint32_t nq, uint32_t nch, uint32_t splits, unsigned long long* partial,
                          cudaStream_t s) {
  if (nch <= 1) return gt_launch<E, M, 1, K>(data, stride, n, queries, nq, nch, splits, partial, s);
  if (nch <= 2) return gt_launch<E, M, 2, K>(data, stride, n, queries, nq, nch, splits, partial, s);
  if (nch <= 4) return gt_launch<E, M, 4, K>(data, stride, n, queries, nq, nch, splits, partial, s);
  if (nch <= 8) return gt_launch<E, M, 8, K>(data, stride, n, queries, nq, nch, splits, partial, s);
  if (nch <= 16) return gt_launch<E, M, 16, K>(data, stride, n, queries, nq, nch, splits, partial, s);
  // wide rows: query rows in shared memory, a point tile beside them
  const uint32_t tile_pts = 16;
  const size_t smem = (size_t(kGtThreads) + tile_pts) * nch * 16;  // <= 227 KB for rows up to 1568 B
  auto kw = gt_wide_kernel<E, M, K>;
  cudaError_t e = cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  dim3 grid((nq + kGtThreads - 1) / kGtThreads, splits);
  kw<<<grid, kGtThreads, smem, s>>>(data, stride, n, queries, nq, nch, splits, tile_pts, partial);
  return cudaGetLastError();
}
template <int E, int M>
cudaError_t gt_dispatch(const uint8_t* data, uint64_t stride, uint64_t n, const uint8_t* queries,
                        uint32_t nq, uint32_t nch, uint32_t k, uint32_t splits, unsigned long long* partial,
                        cudaStream_t s) {
  return k <= 16 ? gt_dispatch_k<E, M, 16>(data, stride, n, queries, nq, nch, splits, partial, s)
                 : gt_dispatch_k<E, M, kGtMaxK>(data, stride, n, queries, nq, nch, splits, partial, s);
}

}  // namespace

cudaError_t launch_choose_start(const uint8_t* data, uint64_t stride, uint64_t n, uint32_t d,
                                int elem, int metric, double* colsum, float* centroid,
                                unsigned long long* best, cudaStream_t s) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(colsum, 0, sizeof(double) * d, s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(best, 0xFF, sizeof(unsigned long long), s)) != cudaSuccess) return e;
  const uint32_t cb = static_cast<uint32_t>((n + 511) / 512);
  const uint32_t ct = d < 256 ? ((d + 31) / 32) * 32 : 256;
  if (elem == kU8) colsum_kernel<kU8><<<cb, ct, 0, s>>>(data, stride, n, d, colsum);
  else if (elem == kI8) colsum_kernel<kI8><<<cb, ct, 0, s>>>(data, stride, n, d, colsum);
  else colsum_kernel<kF32><<<cb, ct, 0, s>>>(data, stride, n, d, colsum);
  centroid_kernel<<<1, 256, 0, s>>>(colsum, n, d, centroid);
  const uint32_t db = static_cast<uint32_t>((n + 255) / 256);
  const size_t smem = sizeof(float) * d;
#define GANN_SD(E, M) start_dist_kernel<E, M><<<db, 256, smem, s>>>(data, stride, n, d, centroid, best)
  if (metric == kL2) {
    if (elem == kU8) GANN_SD(kU8, kL2); else if (elem == kI8) GANN_SD(kI8, kL2); else GANN_SD(kF32, kL2);
  } else {
    if (elem == kU8) GANN_SD(kU8, kIP); else if (elem == kI8) GANN_SD(kI8, kIP); else GANN_SD(kF32, kIP);
  }
#undef GANN_SD
  return cudaGetLastError();
}

void preload_misc(int elem, int metric) {
  touch_kernel(centroid_kernel);
#define GANN_PL(E, M) (touch_kernel(colsum_kernel<E>), touch_kernel(start_dist_kernel<E, M>))
  if (metric == kL2) {
    if (elem == kU8) GANN_PL(kU8, kL2); else if (elem == kI8) GANN_PL(kI8, kL2); else GANN_PL(kF32, kL2);
  } else {
    if (elem == kU8) GANN_PL(kU8, kIP); else if (elem == kI8) GANN_PL(kI8, kIP); else GANN_PL(kF32, kIP);
  }
#undef GANN_PL
}

// Phi^-1(p): Acklam's rational approximation (relative error < 1.2e-9)
// refined by one Halley step on erfc, i.e. to about double precision.
static double norm_ppf(double p) {
  static const double a[6] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                              1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[5] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                              6.680131188771972e+01, -1.328068155288572e+01};
  static const double c[6] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                              -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00};
  static const double d[4] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                              3.754408661907416e+00};
  const double plow = 0.02425;
  double x;
  if (p < plow) {
    const double q = std::sqrt(-2.0 * std::log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else if (p <= 1.0 - plow) {
    const double q = p - 0.5, r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  } else {
    const double q = std::sqrt(-2.0 * std::log(1.0 - p));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  const double e = 0.5 * std::erfc(-x / std::sqrt(2.0)) - p;
  const double u = e * std::sqrt(2.0 * 3.14159265358979323846) * std::exp(x * x / 2.0);
  return x - u / (1.0 + x * u / 2.0);
}

// table[u] = Phi^-1((u + 1/2) / 2^16) on a 2^-16 grid (the grid makes the
// table immune to last-ulp differences between libm builds).
void normal_table(float* out) {
  for (uint32_t u = 0; u < 65536; u++) {
    const double z = norm_ppf((static_cast<double>(u) + 0.5) / 65536.0);
    out[u] = static_cast<float>(std::nearbyint(z * 65536.0) / 65536.0);
  }
}

// The table in device memory, uploaded once per device (read-only).
const float* device_normal_table() {
  static std::mutex mu;
  static float* tabs[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!tabs[dev]) {
    std::vector<float> h(65536);
    normal_table(h.data());
    float* p = nullptr;
    if (cudaMalloc(&p, 65536 * sizeof(float)) != cudaSuccess) return nullptr;
    if (cudaMemcpy(p, h.data(), 65536 * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaFree(p);
      return nullptr;
    }
    tabs[dev] = p;
  }
  return tabs[dev];
}

cudaError_t launch_generate_u8(uint8_t* out, uint64_t out_stride, uint64_t n, uint32_t d,
                               uint32_t clusters, float sigma, float noise_frac,
                               uint64_t center_seed, uint64_t stream_seed, uint64_t row0,
                               cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint32_t thr = static_cast<uint32_t>(static_cast<double>(noise_frac) * 16777216.0);
  const float* tab = device_normal_table();
  if (!tab) return cudaErrorMemoryAllocation;
  gen_u8_kernel<<<148 * 16, 256, 0, s>>>(out, out_stride, n, d, clusters, sigma, thr, center_seed,
                                         stream_seed, row0, tab);
  return cudaGetLastError();
}

cudaError_t launch_generate_f32(float* out, uint64_t n, uint32_t d, uint32_t clusters, float sigma,
                                float norm_sigma, float shift, uint64_t center_seed, uint64_t stream_seed,
                                uint64_t row0, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const float* tab = device_normal_table();
  if (!tab) return cudaErrorMemoryAllocation;
  gen_f32_kernel<<<148 * 16, 256, 0, s>>>(out, n, d, clusters, sigma, norm_sigma, shift, center_seed, stream_seed,
                                          row0, tab);
  return cudaGetLastError();
}

uint32_t groundtruth_splits(uint64_t n, uint32_t nq) {
  const uint32_t qb = (nq + kGtThreads - 1) / kGtThreads;
  uint32_t s = (148 * 8 + qb - 1) / qb;
  s = std::max<uint32_t>(1, std::min<uint32_t>(s, 256));
  while (s > 1 && n / s < 4096) s--;
  return s;
}

cudaError_t launch_groundtruth(const uint8_t* data, uint64_t stride, uint64_t n,
                               const uint8_t* queries, uint32_t nq, uint32_t k, int elem,
                               int metric, uint32_t nch, unsigned long long* partial,
                               uint32_t splits, uint32_t* ids, float* dists, cudaStream_t s) {
  if (nq == 0) return cudaSuccess;
  cudaError_t e;
#define GANN_GT(E, M) e = gt_dispatch<E, M>(data, stride, n, queries, nq, nch, k, splits, partial, s)
  if (metric == kL2) {
    if (elem == kU8) GANN_GT(kU8, kL2); else if (elem == kI8) GANN_GT(kI8, kL2); else GANN_GT(kF32, kL2);
  } else {
    if (elem == kU8) GANN_GT(kU8, kIP); else if (elem == kI8) GANN_GT(kI8, kIP); else GANN_GT(kF32, kIP);
  }
#undef GANN_GT
  if (e != cudaSuccess) return e;
  if (k <= 16)
    gt_merge_kernel<16><<<(nq + 127) / 128, 128, 0, s>>>(partial, nq, splits, k, ids, dists);
  else
    gt_merge_kernel<kGtMaxK><<<(nq + 127) / 128, 128, 0, s>>>(partial, nq, splits, k, ids, dists);
  return cudaGetLastError();
}


// ---- graph row validation ----------------------------------------------------
// The reference's set_neighbors checks (src/graph.cpp:42-59: id in range, no
// self loop) plus its graph invariant of distinct neighbours
// (check_graph_invariants, src/graph.cpp:80-92), and our padding rule (ids
// first, then GANN_NONE). One warp per row; the first bad row (lowest index)
// wins: bad = min(row << 3 | code).
namespace {
__global__ void validate_rows_kernel(const uint32_t* adj, uint64_t rows, uint32_t R, uint64_t n, uint64_t row0,
                                     unsigned long long* bad) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t r = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const uint32_t* row = adj + r * R;
    const uint64_t v = row0 + r;
    uint32_t code = 0;
    bool ended = false;
    for (uint32_t t0 = 0; t0 < R; t0 += 32) {
      const uint32_t t = t0 + lane;
      const uint32_t id = t < R ? row[t] : kNone;
      const bool none = id == kNone;
      const uint32_t nb = __ballot_sync(0xFFFFFFFFu, none && t < R);
      const bool after_pad = !none && (ended || (nb & ((1u << lane) - 1u)) != 0);
      if (after_pad) code = max(code, 1u);
      if (!none && id >= n) code = max(code, 2u);
      if (!none && id == v) code = max(code, 3u);
      // duplicates against this chunk's lower lanes and every earlier chunk
      for (uint32_t c0 = 0; c0 <= t0; c0 += 32) {
        const uint32_t other = c0 + lane < R ? row[c0 + lane] : kNone;
        for (int j = 0; j < 32; j++) {
          const uint32_t o = __shfl_sync(0xFFFFFFFFu, other, j);
          if (!none && o == id && (c0 < t0 || j < lane)) code = max(code, 4u);
        }
      }
      ended = ended || nb != 0;
    }
    code = __reduce_max_sync(0xFFFFFFFFu, code);
    if (lane == 0 && code) atomicMin(bad, (static_cast<unsigned long long>(r) << 3) | code);
  }
}
}  // namespace

cudaError_t launch_validate_rows(const uint32_t* adj, uint64_t rows, uint32_t R, uint64_t n, uint64_t row0,
                                 unsigned long long* bad, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), s);
  if (e != cudaSuccess || rows == 0 || R == 0) return e;
  const uint64_t blocks = std::min<uint64_t>((rows + 7) / 8, 148ull * 16);
  validate_rows_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(adj, rows, R, n, row0, bad);
  return cudaGetLastError();
}

// Stable LSD radix sort of (key, value) u32 pairs over the low `bits` key
// bits (CUB): the semisort for groups too large for the counting group-by's
// in-block ordinal sort. `tmp` is grown as needed (caller-owned).
cudaError_t stable_sort_pairs_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                                  uint32_t* vals_out, uint64_t m, int bits, void** tmp, size_t* tmp_bytes,
                                  cudaStream_t s) {
  size_t need = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, need, keys_in, keys_out, vals_in, vals_out,
                                                  static_cast<int64_t>(m), 0, bits, s);
  if (e != cudaSuccess) return e;
  if (need > *tmp_bytes) {
    if (*tmp) cudaFree(*tmp);
    *tmp = nullptr;
    *tmp_bytes = 0;
    if ((e = cudaMalloc(tmp, need)) != cudaSuccess) return e;
    *tmp_bytes = need;
  }
  return cub::DeviceRadixSort::SortPairs(*tmp, need, keys_in, keys_out, vals_in, vals_out, static_cast<int64_t>(m), 0,
                                         bits, s);
}

// ---- std::shuffle's result from its swap log --------------------------------
// libstdc++'s std::shuffle over n elements is the swap sequence
//   for i = 1 .. n-1: swap(a[i], a[r_i]),  r_i <= i drawn from the generator
// (bits/stl_algo.h; the host records r with an iterator that logs the swaps
// instead of doing them: gann.cu shuffle_swap_log). On iota, a[i] is untouched
// before step i, so step i places value i at position r_i and moves that
// position's occupant to position i. With T_p = the steps that target p in
// ascending order (r_0 := 0 makes 0 the first step of T_0):
//   * the final occupant of p is the last step of T_p, or, when nothing
//     targets p, the first occupant of p;
//   * the first occupant of p (at time p) is the occupant of r_p just before
//     step p: the step before p in T_{r_p}, or, when p is that list's first
//     step, the first occupant of r_p (r_p < p: the chain walks down).
// The lists come from one stable radix sort of (r_i, i); a thread per
// position then follows its chain (expected length O(log n)).
namespace {
__global__ void iota_kernel(uint32_t* v, uint64_t n) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = static_cast<uint32_t>(i);
}
// sorted by target: prev[step] = the step before it on the same target (kNone: first), last[target] = its last step
__global__ void shuffle_lists_kernel(const uint32_t* tgt, const uint32_t* step, uint64_t n, uint32_t* prev,
                                     uint32_t* last) {
  const uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  const uint32_t t = tgt[j], st = step[j];
  prev[st] = (j > 0 && tgt[j - 1] == t) ? step[j - 1] : kNone;
  if (j + 1 == n || tgt[j + 1] != t) last[t] = st;
}
__global__ void shuffle_resolve_kernel(const uint32_t* r, const uint32_t* prev, const uint32_t* last, uint64_t n,
                                       uint32_t* out, uint32_t front, uint32_t* front_pos) {
  const uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (p >= n) return;
  uint32_t v = last[p];
  if (v == kNone) {
    uint32_t q = static_cast<uint32_t>(p);
    while ((v = prev[q]) == kNone) q = r[q];
  }
  out[p] = v;
  if (v == front) *front_pos = static_cast<uint32_t>(p);
}
// shuffled_order's last step (src/builder_common.cpp:104-105): the front vertex swaps into slot 0
__global__ void shuffle_front_kernel(uint32_t* out, const uint32_t* front_pos) {
  const uint32_t p = *front_pos, a = out[0];
  out[0] = out[p];
  out[p] = a;
}
}  // namespace

// out[0..n) = the shuffled insertion order for the swap log r (device, r[0] = 0), with `front` moved to slot 0.
// work: 4 n u32 of scratch (device).
cudaError_t launch_shuffle_from_log(const uint32_t* r, uint64_t n, uint32_t front, uint32_t* work, uint32_t* out,
                                    void** tmp, size_t* tmp_bytes, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  uint32_t* iota = work;
  uint32_t* tgt = work + n;
  uint32_t* step = work + 2 * n;
  uint32_t* prev = work + 3 * n;
  uint32_t* last = iota;  // iota is dead after the sort
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  iota_kernel<<<blocks, 256, 0, s>>>(iota, n);
  int bits = 1;
  while (bits < 32 && (uint64_t(1) << bits) < n) bits++;
  cudaError_t e = stable_sort_pairs_u32(r, tgt, iota, step, n, bits, tmp, tmp_bytes, s);
  if (e != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(last, 0xFF, n * 4, s)) != cudaSuccess) return e;
  shuffle_lists_kernel<<<blocks, 256, 0, s>>>(tgt, step, n, prev, last);
  // the sorted targets are dead once the lists are built: tgt[0] holds front's position
  shuffle_resolve_kernel<<<blocks, 256, 0, s>>>(r, prev, last, n, out, front, tgt);
  shuffle_front_kernel<<<1, 1, 0, s>>>(out, tgt);
  return cudaGetLastError();
}

GANN_CHECK_READER(check_line_misc)

}  // namespace gann
