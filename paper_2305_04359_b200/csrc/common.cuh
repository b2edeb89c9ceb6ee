// common.cuh — device building blocks shared by the gann kernels (sm_100a).
//
// Keys. Every ordered quantity on the path is a (dist: f32, id: u32) pair
// compared lexicographically (neighbor_less, include/graphann/core.hpp:42-44).
// We pack it into one u64: the high word is the f32 mapped to an
// order-preserving u32 (after turning -0.0 into +0.0, which the reference's
// `<` treats as equal), the low word is the id. A single u64 compare is then
// exactly neighbor_less.
//
// Rows. Points live in HBM as rows padded to a multiple of 16 bytes (zero
// fill), so every row is a whole number of 16-byte chunks and can be gathered
// with 128-bit loads. A row of nch chunks is processed by LPR lanes (a power
// of two <= 32), each lane owning chunks sub, sub+LPR, ... (at most CPL of
// them); 32/LPR rows are processed per warp pass and the LPR partial sums are
// combined with xor-shuffles. Zero padding contributes 0 to both L2 and IP.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gann {

// Checked builds (-DGANN_CHECKED, tools/build_variant.sh; the GPU test
// tests/test_gpu_checked.py): index bounds of the kernels' shared-memory and
// output writes are tested on the device; a failure records its source line
// (the largest failing line wins) instead of writing out of bounds, and
// gann_debug_check_line() reports it. compute-sanitizer is not available on
// the GPU pool, so this is the memory-safety evidence. Release builds compile
// the checks away.
#ifdef GANN_CHECKED
static __device__ unsigned int g_check_line = 0;
#define GANN_CHECK(c)                                         \
  do {                                                        \
    if (!(c)) atomicMax(&::gann::g_check_line, __LINE__);     \
  } while (0)
#define GANN_CHECKED_ONLY(x) x
// a translation unit's reader: the largest failing line, then cleared
#define GANN_CHECK_READER(name)                                   \
  unsigned name() {                                               \
    unsigned v = 0, z = 0;                                        \
    cudaMemcpyFromSymbol(&v, ::gann::g_check_line, sizeof(v));    \
    cudaMemcpyToSymbol(::gann::g_check_line, &z, sizeof(z));      \
    return v;                                                     \
  }
#else
#define GANN_CHECK_READER(name) \
  unsigned name() { return 0; }
#define GANN_CHECK(c) \
  do {                \
  } while (0)
#define GANN_CHECKED_ONLY(x)
#endif

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint64_t kMaxKey = 0xFFFFFFFFFFFFFFFFull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  // splitmix64 finaliser — include/graphann/core.hpp:47-53
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t a, uint64_t b) {
  return mix64(a ^ mix64(b));
}

__device__ __forceinline__ uint32_t f2ord(float d) {
  uint32_t b = __float_as_uint(__fadd_rn(d, 0.0f));  // -0.0 -> +0.0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
  uint32_t b = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  return __uint_as_float(b);
}
__device__ __forceinline__ uint64_t make_key(float d, uint32_t id) {
  return (static_cast<uint64_t>(f2ord(d)) << 32) | id;
}
__device__ __forceinline__ float key_dist(uint64_t k) { return ord2f(static_cast<uint32_t>(k >> 32)); }
__device__ __forceinline__ uint32_t key_id(uint64_t k) { return static_cast<uint32_t>(k); }

__device__ __forceinline__ uint4 ldg_nc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ---- distance arithmetic -------------------------------------------------
// src/metric.cpp:38-59. Integer element kinds are exact in int32 (the
// reference accumulates in int32 and casts to float once); f32 uses FMA
// partial sums, which differ from the reference's sequential float sum only
// in the last ulps (tolerance stated by the north star: 1e-5 relative).
enum Elem { kU8 = 0, kI8 = 1, kF32 = 2 };
enum MetricKind { kL2 = 0, kIP = 1 };

template <int E, int M>
struct DistOp;

template <>
struct DistOp<kU8, kL2> {
  using acc_t = uint32_t;
  static __device__ __forceinline__ acc_t zero() { return 0u; }
  static __device__ __forceinline__ acc_t chunk(const uint4& a, const uint4& b, acc_t acc) {
    uint32_t t;
    t = __vabsdiffu4(a.x, b.x); acc = __dp4a(t, t, acc);
    t = __vabsdiffu4(a.y, b.y); acc = __dp4a(t, t, acc);
    t = __vabsdiffu4(a.z, b.z); acc = __dp4a(t, t, acc);
    t = __vabsdiffu4(a.w, b.w); acc = __dp4a(t, t, acc);
    return acc;
  }
  static __device__ __forceinline__ float finish(acc_t a) { return __int2float_rn(static_cast<int>(a)); }
};
template <>
struct DistOp<kI8, kL2> {
  using acc_t = uint32_t;
  static __device__ __forceinline__ acc_t zero() { return 0u; }
  static __device__ __forceinline__ acc_t chunk(const uint4& a, const uint4& b, acc_t acc) {
    uint32_t t;
    t = __vabsdiffs4(a.x, b.x); acc = __dp4a(t, t, acc);
    t = __vabsdiffs4(a.y, b.y); acc = __dp4a(t, t, acc);
    t = __vabsdiffs4(a.z, b.z); acc = __dp4a(t, t, acc);
    t = __vabsdiffs4(a.w, b.w); acc = __dp4a(t, t, acc);
    return acc;
  }
  static __device__ __forceinline__ float finish(acc_t a) { return __int2float_rn(static_cast<int>(a)); }
};
template <>
struct DistOp<kU8, kIP> {
  using acc_t = uint32_t;
  static __device__ __forceinline__ acc_t zero() { return 0u; }
  static __device__ __forceinline__ acc_t chunk(const uint4& a, const uint4& b, acc_t acc) {
    acc = __dp4a(a.x, b.x, acc);
    acc = __dp4a(a.y, b.y, acc);
    acc = __dp4a(a.z, b.z, acc);
    acc = __dp4a(a.w, b.w, acc);
    return acc;
  }
  static __device__ __forceinline__ float finish(acc_t a) { return -__int2float_rn(static_cast<int>(a)); }
};
template <>
struct DistOp<kI8, kIP> {
  using acc_t = int;
  static __device__ __forceinline__ acc_t zero() { return 0; }
  static __device__ __forceinline__ acc_t chunk(const uint4& a, const uint4& b, acc_t acc) {
    acc = __dp4a(static_cast<int>(a.x), static_cast<int>(b.x), acc);
    acc = __dp4a(static_cast<int>(a.y), static_cast<int>(b.y), acc);
    acc = __dp4a(static_cast<int>(a.z), static_cast<int>(b.z), acc);
    acc = __dp4a(static_cast<int>(a.w), static_cast<int>(b.w), acc);
    return acc;
  }
  static __device__ __forceinline__ float finish(acc_t a) { return -__int2float_rn(a); }
};
template <>
struct DistOp<kF32, kL2> {
  using acc_t = float;
  static __device__ __forceinline__ acc_t zero() { return 0.0f; }
  static __device__ __forceinline__ acc_t chunk(const uint4& a, const uint4& b, acc_t acc) {
    float d;
    d = __uint_as_float(a.x) - __uint_as_float(b.x); acc = fmaf(d, d, acc);
    d = __uint_as_float(a.y) - __uint_as_float(b.y); acc = fmaf(d, d, acc);
    d = __uint_as_float(a.z) - __uint_as_float(b.z); acc = fmaf(d, d, acc);
    d = __uint_as_float(a.w) - __uint_as_float(b.w); acc = fmaf(d, d, acc);
    return acc;
  }
  static __device__ __forceinline__ float finish(acc_t a) { return a; }
};
template <>
struct DistOp<kF32, kIP> {
  using acc_t = float;
  static __device__ __forceinline__ acc_t zero() { return 0.0f; }
  static __device__ __forceinline__ acc_t chunk(const uint4& a, const uint4& b, acc_t acc) {
    acc = fmaf(__uint_as_float(a.x), __uint_as_float(b.x), acc);
    acc = fmaf(__uint_as_float(a.y), __uint_as_float(b.y), acc);
    acc = fmaf(__uint_as_float(a.z), __uint_as_float(b.z), acc);
    acc = fmaf(__uint_as_float(a.w), __uint_as_float(b.w), acc);
    return acc;
  }
  static __device__ __forceinline__ float finish(acc_t a) { return -a; }
};

template <int LPR, typename T>
__device__ __forceinline__ T group_sum(T v) {
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// Lower bound of key k in sorted a[0..n): first index with a[i] >= k.
__device__ __forceinline__ uint32_t lower_bound_u64(const uint64_t* a, uint32_t n, uint64_t k) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < k) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// lower_bound_u64 without data-dependent branches: the count of entries < k,
// found by power-of-two steps (floor(log2 n) + 1 probes, one LDS each).
__device__ __forceinline__ uint32_t lower_bound_steps_u64(const uint64_t* a, uint32_t n, uint64_t k) {
  uint32_t pos = 0;
  for (uint32_t step = n ? 1u << (31 - __clz(n)) : 0u; step; step >>= 1) {
    const uint32_t j = pos + step;
    if (j <= n && a[j - 1] < k) pos = j;
  }
  return pos;
}

// Sum U per-lane partials over the LPR lanes of a row group so that lane
// (sub mod U) ends up holding the total of row `sub mod U` (U <= LPR, both
// powers of two): plain butterflies for the lane bits above U, then a
// transposed butterfly that halves the live values each step — LPR=U=8 costs
// 4+2+1 shuffles for 8 rows instead of 3 per row.
template <int LPR, int U, typename T>
__device__ __forceinline__ T transpose_reduce(T (&v)[U], int sub) {
#pragma unroll
  for (int o = LPR / 2; o >= U; o >>= 1) {
#pragma unroll
    for (int u = 0; u < U; u++) v[u] += __shfl_xor_sync(0xFFFFFFFFu, v[u], o);
  }
#pragma unroll
  for (int w = U / 2; w >= 1; w >>= 1) {
    const bool hi = (sub & w) != 0;
#pragma unroll
    for (int i = 0; i < w; i++) {
      const T send = hi ? v[i] : v[i + w];
      const T keep = hi ? v[i + w] : v[i];
      v[i] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, w);
    }
  }
  return v[0];
}

}  // namespace gann
