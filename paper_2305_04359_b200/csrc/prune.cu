// prune.cu — robustPrune (alpha_prune) for many lists at once, one CTA per list.
//
// Behaviour contract: graphann::alpha_prune (src/prune.cpp:8-44):
// drop p, sort the candidates by (dist, id), then walk them in order; a
// candidate that is still alive is selected, and unless its distance is 0 it
// culls every later alive candidate j with alpha*d(sel, j) <= d(p, j)
// (scale_candidate) or d(sel, j) < alpha*d(p, sel) (scale_selected); stop at R.
//
// GPU shape. The candidate keys sit in shared memory and are bitonic-sorted
// by the CTA. The alive list is a compacted index array in key order; every
// selection computes its distances to all alive candidates in parallel (LPR
// lanes per row, 16-byte gathers of rows that the preceding search just pulled
// into L2) and stable-compacts the survivors. Each alpha*via is one IEEE f32
// multiply (__fmul_rn) so the comparison is bit-identical to the reference;
// integer distances are exact. 32-thread CTAs serve the insert-time lists
// (|V| ~ L); 256-thread CTAs with up to 16k candidates serve back-edge hubs.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace gann {

size_t prune_smem_bytes(uint32_t mcap, uint32_t R) {
  uint32_t M = 32;
  while (M < mcap && M < (1u << 16)) M <<= 1;
  size_t b = size_t(M) * 8 + 2 * size_t(M) * 2 + size_t(M) + size_t(R) * 4;
  return (b + 15) & ~size_t(15);
}

template <int NT>
__device__ __forceinline__ void cta_sync() {
  if (NT == 32) __syncwarp(); else __syncthreads();
}

// Stable compaction of src[0..n) into dst by flags kf[0..n); returns count.
template <int NT>
__device__ __forceinline__ uint32_t cta_compact(const uint16_t* src, const uint8_t* kf, uint32_t n,
                                                uint16_t* dst, uint32_t* warp_tot) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t total = 0;
  for (uint32_t b0 = 0; b0 < n; b0 += NT) {
    const uint32_t i = b0 + tid;
    const bool keep = i < n && kf[i];
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
    uint32_t off = __popc(bal & ((1u << lane) - 1u));
    if (NT == 32) {
      if (keep) dst[total + off] = src[i];
      total += __popc(bal);
    } else {
      if (lane == 0) warp_tot[w] = __popc(bal);
      __syncthreads();
      uint32_t before = 0, all = 0;
      for (int t = 0; t < NT / 32; t++) {
        const uint32_t c = warp_tot[t];
        if (t < w) before += c;
        all += c;
      }
      if (keep) dst[total + before + off] = src[i];
      total += all;
      __syncthreads();
    }
  }
  return total;
}

template <int E, int M, int LPR, int CPL, int NT>
__global__ void __launch_bounds__(NT) prune_kernel(const PruneArgs a, const uint32_t Mcap) {
  using Op = DistOp<E, M>;
  constexpr int GROUPS = NT / LPR;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t warp_tot[NT / 32];
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  uint16_t* alA = reinterpret_cast<uint16_t*>(keys + Mcap);
  uint16_t* alB = alA + Mcap;
  uint8_t* kf = reinterpret_cast<uint8_t*>(alB + Mcap);
  uint32_t* sel = reinterpret_cast<uint32_t*>(kf + Mcap);
  const int tid = threadIdx.x;
  const int sub = tid & (LPR - 1);
  const int grp = tid / LPR;
  const uint32_t nch = static_cast<uint32_t>(a.stride >> 4);
  const uint32_t R = a.R;

  for (uint32_t li = blockIdx.x; li < a.count; li += gridDim.x) {
    const uint32_t l = a.list_index ? a.list_index[li] : li;
    const uint32_t p = a.points[l];
    uint64_t beg, m;
    beg = a.begins ? a.begins[l] : uint64_t(l) * a.fixed_stride;
    m = a.lengths[l];
    uint32_t* orow = a.out_rows ? a.out_rows + uint64_t(l) * R : a.out_adj + uint64_t(p - a.out_base) * R;
    if (m < a.mmin) continue;  // another launch's bin
    if (m > a.mcap) {  // caller routes long lists elsewhere; never truncate silently
      if (tid == 0 && !a.skip_long) atomicAdd(a.too_long, 1u);
      continue;
    }
    uint32_t Mp = 32;
    while (Mp < m) Mp <<= 1;
    for (uint32_t i = tid; i < Mp; i += NT) {
      uint64_t k = kMaxKey;
      if (i < m) {
        const uint32_t id = a.cand_ids[beg + i];
        if (id != p) k = make_key(a.cand_dists[beg + i], id);  // prune.cpp:18-20 drops p
      }
      keys[i] = k;
    }
    cta_sync<NT>();
    // bitonic sort by (dist, id) — prune.cpp:21
    for (uint32_t k = 2; k <= Mp; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = tid; i < Mp; i += NT) {
          const uint32_t ixj = i ^ j;
          if (ixj > i) {
            const uint64_t x = keys[i], y = keys[ixj];
            const bool up = (i & k) == 0;
            if ((x > y) == up) {
              keys[i] = y;
              keys[ixj] = x;
            }
          }
        }
        cta_sync<NT>();
      }
    }
    const uint32_t m2 = lower_bound_u64(keys, Mp, kMaxKey);
    for (uint32_t i = tid; i < m2; i += NT) alA[i] = static_cast<uint16_t>(i);
    cta_sync<NT>();

    uint16_t* alive = alA;
    uint32_t nalive = m2, nsel = 0;
    uint64_t evals = 0;
    while (nsel < R && nalive > 0) {  // prune.cpp:25-43
      const uint64_t sk = keys[alive[0]];
      if (tid == 0) sel[nsel] = key_id(sk);
      nsel++;
      if (nsel == R) break;
      if (key_dist(sk) == 0.0f) {  // :32 a zero-distance pick culls nothing
        alive++;
        nalive--;
        continue;
      }
      const uint32_t sid = key_id(sk);
      const float sdist = key_dist(sk);
      uint4 sr[CPL];
      const uint8_t* srow = a.data + uint64_t(sid) * a.stride;
#pragma unroll
      for (int c = 0; c < CPL; c++) {
        const uint32_t ch = sub + c * LPR;
        sr[c] = ch < nch ? __ldg(reinterpret_cast<const uint4*>(srow) + ch) : make_uint4(0, 0, 0, 0);
      }
      const uint32_t rest = nalive - 1;  // candidates after the selection
      evals += rest;
      constexpr int U = 4;
      for (uint32_t b0 = 0; b0 < rest; b0 += GROUPS * U) {
        uint4 x[U][CPL];
        uint32_t idx[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const uint32_t t = b0 + u * GROUPS + grp;
          idx[u] = t < rest ? alive[1 + t] : 0xFFFFu;
          const uint32_t id = t < rest ? key_id(keys[idx[u]]) : 0u;
          const uint8_t* rp = a.data + uint64_t(id) * a.stride;
#pragma unroll
          for (int c = 0; c < CPL; c++) {
            const uint32_t ch = sub + c * LPR;
            x[u][c] = (t < rest && ch < nch) ? __ldg(reinterpret_cast<const uint4*>(rp) + ch)
                                             : make_uint4(0, 0, 0, 0);
          }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
          typename Op::acc_t acc = Op::zero();
#pragma unroll
          for (int c = 0; c < CPL; c++) acc = Op::chunk(sr[c], x[u][c], acc);
          acc = group_sum<LPR>(acc);
          const uint32_t t = b0 + u * GROUPS + grp;
          if (sub == 0 && t < rest) {
            const float via = Op::finish(acc);
            const float dj = key_dist(keys[idx[u]]);
            // prune.cpp:37-39, one IEEE multiply, never contracted
            const bool drop = a.rule == 0 ? (__fmul_rn(a.alpha, via) <= dj)
                                          : (via < __fmul_rn(a.alpha, sdist));
            kf[t] = drop ? 0 : 1;
          }
        }
      }
      cta_sync<NT>();
      uint16_t* dst = (alive >= alA && alive < alA + Mcap) ? alB : alA;
      nalive = cta_compact<NT>(alive + 1, kf, rest, dst, warp_tot);
      alive = dst;
      cta_sync<NT>();
    }
    cta_sync<NT>();
    for (uint32_t i = tid; i < R; i += NT) orow[i] = i < nsel ? sel[i] : kNone;
    if (tid == 0) {
      if (a.n_out) a.n_out[l] = nsel;
      if (a.spre && !a.out_rows) a.spre[p - a.out_base] = static_cast<uint8_t>(nsel < 255 ? nsel : 255);
      if (a.stats) {
        atomicAdd(stat_slot(a.stats) + kStPruneLists, 1ull);
        atomicAdd(stat_slot(a.stats) + kStPruneCands, static_cast<unsigned long long>(m));
        atomicAdd(stat_slot(a.stats) + kStPruneEvals, static_cast<unsigned long long>(evals));
      }
    }
    cta_sync<NT>();
  }
}

// ---- integer lists on the tensor cores ---------------------------------------
// For u8/i8 rows every distance the greedy needs is an exact int32:
// d(i, j) = |x_i|^2 + |x_j|^2 - 2 x_i.x_j (L2) or -x_i.x_j (IP), identical to
// the reference's sequential int32 sum. The candidates' rows are gathered
// once into shared memory (sorted order, rows padded to 32-byte k-steps,
// stride Kp+16 so ldmatrix is bank-conflict free) and the Gram entries come
// from int8 MMA (mma.sync m16n8k32 s32 += u8/s8 x u8/s8, fragments loaded with
// ldmatrix). The distance rows are produced lazily, one 16-row block at a time
// as the greedy walk enters it (columns right of the block only), so shared
// memory holds 16 x mc distances instead of mc x mc, and the walk itself
// reads distances instead of gathering rows.
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}

template <bool SIGNED>
__device__ __forceinline__ void mma_i8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if (SIGNED)
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  else
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

struct MmaLayout {
  uint32_t mc;   // max candidates (32 * W)
  uint32_t kp;   // row bytes rounded up to 32
  uint32_t xs;   // smem row stride (kp + 16, ldmatrix bank-conflict free)
  uint32_t w;    // 32-bit words per cull mask
  uint32_t stride;  // words per list in the global hand-off region
  size_t off_sk, off_perm, off_x, off_xp, off_norm, off_dk, off_ns, off_cm, total;
};
__host__ __device__ inline MmaLayout mma_layout(uint32_t mcap, uint32_t stride, uint32_t /*R*/) {
  MmaLayout l;
  l.w = mcap <= 128 ? 4 : (mcap <= 256 ? 8 : 16);
  // short lists (re-prunes: a row of R plus a few sources) get a smaller
  // staging area, so more CTAs fit an SM; the mask rows stay W words
  l.mc = ((mcap < l.w * 32 ? mcap : l.w * 32) + 15) & ~15u;
  l.kp = (stride + 31) & ~31u;
  l.xs = l.kp + 16;
  l.stride = 4 + l.mc + l.w + l.mc * l.w;  // [m2, pad x3][ids mc][zero mask W][cull rows mc*W]
  size_t o = size_t(l.mc) * 8;              // input-order keys
  l.off_sk = o;
  o += size_t(l.mc) * 8;                    // sorted keys
  l.off_perm = o;
  o += size_t(l.mc) * 2;
  o = (o + 15) & ~size_t(15);
  l.off_x = o;
  o += size_t(l.mc + 1) * l.xs;             // + one zero row for padding tiles
  l.off_xp = o;
  o += l.xs;
  l.off_norm = o;
  o += size_t(l.mc + 1) * 4;
  l.off_dk = o;                              // sorted norms (int)
  o += size_t(l.mc + 16) * 4;
  l.off_ns = o;                              // sorted cull thresholds (int)
  o += size_t(l.mc + 16) * 4;
  o = (o + 15) & ~size_t(15);
  l.off_cm = o;
  o += size_t(l.mc) * l.w * 4 + size_t(l.w) * 4;
  l.total = (o + 15) & ~size_t(15);
  return l;
}

#ifndef GANN_PREP_GU
#define GANN_PREP_GU 4  // candidate rows in flight per thread in the prep gather
#endif

// Stage-1 -> stage-2 hand-off buffer (grows; one per process and device).
constexpr uint64_t kHandoffMax = 1ull << 30;  // launches are chunked to fit

void prune_release(PruneHandoff* h, cudaStream_t s) {
  if (!h || !h->buf) return;
  cudaStreamSynchronize(s);
  cudaFree(h->buf);
  h->buf = nullptr;
  h->cap = 0;
}

// The index's hand-off region, grown to `bytes`. Only the owning index's
// stream uses it, so a regrowth needs to wait for that stream alone.
uint32_t* prune_handoff(PruneHandoff* h, uint64_t bytes, cudaStream_t s) {
  if (!h) return nullptr;
  if (bytes > h->cap) {
    // grows geometrically (a build's lists per launch double batch by batch;
    // every regrowth is a stream sync + a large cudaMalloc)
    const uint64_t want = std::max<uint64_t>(bytes, std::min<uint64_t>(2 * h->cap, kHandoffMax));
    cudaStreamSynchronize(s);
    if (h->buf) cudaFree(h->buf);
    h->buf = nullptr;
    h->cap = 0;
    if (cudaMalloc(&h->buf, want) != cudaSuccess) return nullptr;
    h->cap = want;
  }
  return h->buf;
}

// Stage 1 of the integer prune (one CTA per list, no serial part): gather the
// candidates' rows once into shared memory; when the caller has no distances
// (back-edge re-prunes) compute d(p, .) from the same rows; rank-sort the
// (dist, id) keys; evaluate every cull test of the upper triangle from IMMA
// Gram tiles (rows addressed through the sort permutation); hand the sorted
// ids and the cull bitmasks to stage 2 through global memory.
//
// The greedy of prune.cpp:25-43 needs, for a selected i, the test "i culls j"
// only for later j, and its outcome does not depend on which candidates are
// still alive — so evaluating all of them up front is exact.
// Largest integer S with pred(S), pred monotone (true up to a point, then
// false) over [-2^30, 2^30]; e is an estimate of the answer. Exponential
// search from e, then bisection: a few evaluations when e is close.
template <class Pred>
__device__ __forceinline__ int last_true(Pred pred, float e) {
  constexpr int kLo = -(1 << 30), kHi = 1 << 30;
  const int e0 = e != e ? 0 : static_cast<int>(fminf(fmaxf(floorf(e), float(kLo)), float(kHi)));
  int lo, hi;  // pred(lo) true (or lo = kLo - 1), pred(hi) false (or hi = kHi + 1)
  if (pred(e0)) {
    lo = e0;
    int st = 1;
    hi = e0;
    while (true) {
      const long long c = static_cast<long long>(lo) + st;
      if (c > kHi) { hi = kHi + 1; break; }
      if (!pred(static_cast<int>(c))) { hi = static_cast<int>(c); break; }
      lo = static_cast<int>(c);
      st <<= 1;
    }
  } else {
    hi = e0;
    int st = 1;
    while (true) {
      const long long c = static_cast<long long>(hi) - st;
      if (c < kLo) { lo = kLo - 1; break; }
      if (pred(static_cast<int>(c))) { lo = static_cast<int>(c); break; }
      hi = static_cast<int>(c);
      st <<= 1;
    }
  }
  while (hi - lo > 1) {
    const int mid = lo + (hi - lo) / 2;
    if (pred(mid)) lo = mid; else hi = mid;
  }
  return lo;
}

// Threads per CTA by mask width (measured at c1): 96 for the short lists
// (W = 4, mostly re-prunes of ~70 candidates: -5% against 128, +20% at 64,
// +42% at 256), 256 for the long insert-time lists (W >= 8: -10% against 128).
#ifndef GANN_PREP_NT4
#define GANN_PREP_NT4 96
#endif
#ifndef GANN_PREP_NT8
#define GANN_PREP_NT8 256
#endif
template <int W>
struct PrepThreads {
  static constexpr int value = W >= 8 ? GANN_PREP_NT8 : GANN_PREP_NT4;
};

template <int E, int M, int W, int RULE>
__global__ void __launch_bounds__(PrepThreads<W>::value)
    prune_prep_kernel(const PruneArgs a, const MmaLayout ly, uint32_t* hand, uint32_t l0, uint32_t lcount) {
  using Op = DistOp<E, M>;
  constexpr int NT = PrepThreads<W>::value;
  constexpr bool SIGNED = E == kI8;
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* tk = reinterpret_cast<uint64_t*>(smem);
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem + ly.off_sk);
  uint16_t* perm = reinterpret_cast<uint16_t*>(smem + ly.off_perm);
  uint8_t* X = smem + ly.off_x;
  uint8_t* Xp = smem + ly.off_xp;
  int* norm = reinterpret_cast<int*>(smem + ly.off_norm);
  uint32_t* cm = reinterpret_cast<uint32_t*>(smem + ly.off_cm);
  uint32_t* zmask = cm + ly.mc * W;
  int* sn = reinterpret_cast<int*>(smem + ly.off_dk);  // sorted norms
  int* ns = reinterpret_cast<int*>(smem + ly.off_ns);
  __shared__ uint32_t sh_m2, sh_pre;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t mc = ly.mc, xs = ly.xs, kp = ly.kp;
  const uint32_t nch = static_cast<uint32_t>(a.stride >> 4);
  const uint32_t kch = kp >> 4;
  const uint32_t FULL = 0xFFFFFFFFu;
  // the zero row that pads partial tiles (written once)
  for (uint32_t c = tid; c < kch; c += NT) *reinterpret_cast<uint4*>(X + size_t(mc) * xs + c * 16) = make_uint4(0, 0, 0, 0);
  if (tid == 0) norm[mc] = 0;

  // A list's header (index, length, point, offset, verified-prefix length)
  // is loaded up front, one iteration ahead when a CTA takes several lists
  // (one CTA per list measured faster than a resident grid: the CTAs'
  // phases overlap better than one CTA's consecutive lists).
  struct Head {
    uint32_t l, m, p, spre;
    uint64_t beg;
  };
  auto head = [&](uint32_t rel) {
    Head h{0, 0, 0, 0, 0};
    if (rel >= lcount) return h;
    const uint32_t li = l0 + rel;
    h.l = a.list_index ? a.list_index[li] : li;
    h.m = a.lengths[h.l];
    h.p = a.points[h.l];
    h.beg = a.begins ? a.begins[h.l] : uint64_t(h.l) * a.fixed_stride;
    h.spre = (a.row_lists && a.spre) ? a.spre[h.p - a.out_base] : 0u;
    return h;
  };
  Head nxt = head(blockIdx.x);
  for (uint32_t rel = blockIdx.x; rel < lcount; rel += gridDim.x) {
    const Head cur = nxt;
    nxt = head(rel + gridDim.x);
    const uint32_t m = cur.m;
    if (m < a.mmin || m > a.mcap) continue;  // another launch's bin (the walk skips it too)
    const uint32_t p = cur.p;
    const uint64_t beg = cur.beg;
    uint32_t* out = hand + size_t(rel) * ly.stride;
    __syncthreads();
    if (tid == 0) {
      sh_m2 = 0;
      sh_pre = m;
    }
    for (uint32_t i = tid; i < W; i += NT) zmask[i] = 0u;
    // gather rows in input order (+ p's row when distances must be computed)
    const bool own_d = a.cand_dists == nullptr;
    const uint32_t rows_g = m + (own_d ? 1u : 0u);
    if ((kch & (kch - 1)) == 0 && kch <= NT) {
      // a thread keeps one chunk column; 4 rows' loads in flight per thread
      const uint32_t lk = __ffs(kch) - 1, c = tid & (kch - 1), step = NT >> lk;
      constexpr int GU = GANN_PREP_GU;
      for (uint32_t r0 = tid >> lk; r0 < rows_g; r0 += GU * step) {
        uint4 v[GU];
#pragma unroll
        for (int u = 0; u < GU; u++) {
          const uint32_t r = r0 + u * step;
          const uint32_t id = r < m ? a.cand_ids[beg + r] : p;
          v[u] = (r < rows_g && c < nch) ? __ldg(reinterpret_cast<const uint4*>(a.data + uint64_t(id) * a.stride) + c)
                                         : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < GU; u++) {
          const uint32_t r = r0 + u * step;
          GANN_CHECK(r >= rows_g || r <= mc);
          if (r < rows_g) *reinterpret_cast<uint4*>((r < m ? X + size_t(r) * xs : Xp) + c * 16) = v[u];
        }
      }
    } else {
      for (uint32_t t = tid; t < rows_g * kch; t += NT) {
        const uint32_t r = t / kch, c = t - r * kch;
        const uint32_t id = r < m ? a.cand_ids[beg + r] : p;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (c < nch) v = __ldg(reinterpret_cast<const uint4*>(a.data + uint64_t(id) * a.stride) + c);
        uint8_t* dst = r < m ? X + size_t(r) * xs : Xp;
        *reinterpret_cast<uint4*>(dst + c * 16) = v;
      }
    }
    for (uint32_t t = tid; t < m * (W / 4); t += NT) reinterpret_cast<uint4*>(cm)[t] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    // keys (distances from the caller, or d(p, .) — src/builder_common.cpp:136)
    // and the rows' norms. Re-prunes (d(p, .) computed here, ~70 rows): two
    // threads per row, each summing every other 16-byte chunk, combined with
    // one shuffle (integer sums: exact in any order; -6.5% re-prune time).
    // Insert prunes (up to 3L rows, distances given): one thread per row.
    if (!own_d) {
      for (uint32_t i = tid; i < m; i += NT) {
        const uint32_t id = a.cand_ids[beg + i];
        uint64_t k = kMaxKey;
        if (id != p) {  // prune.cpp:18-20 drops p
          k = make_key(a.cand_dists[beg + i], id);
          atomicAdd(&sh_m2, 1u);
        }
        tk[i] = k;
      }
      for (uint32_t r = tid; r < m; r += NT) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(X + size_t(r) * xs);
        int acc = 0;
        for (uint32_t i = 0; i < (kp >> 2); i++) {
          if (SIGNED) acc = __dp4a(static_cast<int>(w[i]), static_cast<int>(w[i]), acc);
          else acc = static_cast<int>(__dp4a(w[i], w[i], static_cast<uint32_t>(acc)));
        }
        norm[r] = acc;
      }
    }
    for (uint32_t base = 0; own_d && base < m; base += NT / 2) {  // uniform trip count (shuffles inside)
      const uint32_t r = base + (tid >> 1), h = tid & 1;
      int nrm = 0;
      typename Op::acc_t dd = Op::zero();
      if (r < m) {
        for (uint32_t c = h; c < kch; c += 2) {
          const uint4 xv = *reinterpret_cast<const uint4*>(X + size_t(r) * xs + c * 16);
          if (SIGNED) {
            nrm = __dp4a(static_cast<int>(xv.x), static_cast<int>(xv.x), nrm);
            nrm = __dp4a(static_cast<int>(xv.y), static_cast<int>(xv.y), nrm);
            nrm = __dp4a(static_cast<int>(xv.z), static_cast<int>(xv.z), nrm);
            nrm = __dp4a(static_cast<int>(xv.w), static_cast<int>(xv.w), nrm);
          } else {
            uint32_t un = static_cast<uint32_t>(nrm);
            un = __dp4a(xv.x, xv.x, un);
            un = __dp4a(xv.y, xv.y, un);
            un = __dp4a(xv.z, xv.z, un);
            un = __dp4a(xv.w, xv.w, un);
            nrm = static_cast<int>(un);
          }
          if (own_d && c < nch) dd = Op::chunk(*reinterpret_cast<const uint4*>(Xp + c * 16), xv, dd);
        }
      }
      nrm += __shfl_xor_sync(FULL, nrm, 1);
      dd += __shfl_xor_sync(FULL, dd, 1);
      if (r < m && h == 0) {
        norm[r] = nrm;
        const uint32_t id = a.cand_ids[beg + r];
        uint64_t k = kMaxKey;
        if (id != p) {  // prune.cpp:18-20 drops p
          k = make_key(own_d ? Op::finish(dd) : a.cand_dists[beg + r], id);
          atomicAdd(&sh_m2, 1u);
        }
        tk[r] = k;
      }
    }
    __syncthreads();
    // rank sort by (dist, id) — prune.cpp:21 (keys are distinct; p carries
    // kMaxKey and is not written). Re-prune lists are a row in ascending
    // order (a prune's output) with a few sources appended, so: find the
    // longest ascending prefix P, then a prefix key's rank is its index plus
    // the suffix keys below it, and a suffix key's rank is a binary search in
    // the prefix plus the other suffix keys below it (O(m - P) per key).
    // Re-prunes of hubs (a row plus many new sources: a long unsorted tail):
    // a bitonic sort of (key, index) in shared memory replaces the
    // O(m (m - P)) ranking (-7% re-prune time). Insert-time lists keep the
    // ranking: measured, the sort's barriers cost more at |V| ~ 1.3 L.
    for (uint32_t i = tid; i + 1 < m; i += NT)
      if (!(tk[i] < tk[i + 1])) atomicMin(&sh_pre, i + 1);
    __syncthreads();
    const uint32_t P = sh_pre;  // keys [0, P) ascend
    uint32_t Mp = 32;
    while (Mp < m) Mp <<= 1;
    if (own_d && (m - P) * m > 40000u && Mp <= mc) {
      for (uint32_t i = tid; i < Mp; i += NT) {
        sk[i] = i < m ? tk[i] : kMaxKey;
        perm[i] = static_cast<uint16_t>(i);
      }
      __syncthreads();
      for (uint32_t k2 = 2; k2 <= Mp; k2 <<= 1) {
        for (uint32_t j = k2 >> 1; j > 0; j >>= 1) {
          for (uint32_t i = tid; i < Mp; i += NT) {
            const uint32_t ixj = i ^ j;
            if (ixj > i) {
              const uint64_t x = sk[i], y = sk[ixj];
              if ((x > y) == ((i & k2) == 0)) {
                sk[i] = y;
                sk[ixj] = x;
                const uint16_t t = perm[i];
                perm[i] = perm[ixj];
                perm[ixj] = t;
              }
            }
          }
          __syncthreads();
        }
      }
    } else {
      for (uint32_t i = tid; i < m; i += NT) {
        const uint64_t k = tk[i];
        if (k == kMaxKey) continue;
        uint32_t r;
        if (i < P) {
          r = i;
        } else {
          uint32_t lo = 0, hi = P;
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (tk[mid] < k) lo = mid + 1; else hi = mid;
          }
          r = lo;
        }
        for (uint32_t j = P; j < m; j++) r += tk[j] < k ? 1u : 0u;
        sk[r] = k;
        perm[r] = static_cast<uint16_t>(i);
      }
    }
    __syncthreads();
    const uint32_t m2 = sh_m2;
    const uint32_t mpad = (m2 + 15) & ~15u;
    const uint32_t mw = (m2 + 31) >> 5;
    // per sorted position: the cull thresholds. With S(i, j) the exact int
    // the reference converts (L2: |x_i|^2 + |x_j|^2 - 2 x_i.x_j; IP: -x_i.x_j),
    // prune.cpp:37-39 culls j from pick i iff
    //   rule 0: fmul(alpha, float(S)) <= d(p, j)  <=>  S <= T_j
    //   rule 1: float(S) < fmul(alpha, d(p, i))   <=>  S <= V_i
    // both monotone in S, so T_j / V_i are exact. Stored folded with the
    // norms: thr[j] = T_j - |x_j|^2 (rule 0, per column) or V_i - |x_i|^2
    // (rule 1, per row); padding positions never cull.
    for (uint32_t i = tid; i < mpad; i += NT) {
      int th = -(1 << 30);
      int nrm = 0;
      if (i < m2) {
        const float dd = key_dist(sk[i]);
        nrm = M == kL2 ? norm[perm[i]] : 0;
        const float alpha = a.alpha;
        if (RULE == 0)
          th = last_true([&](int S) { return __fmul_rn(alpha, __int2float_rn(S)) <= dd; }, dd / alpha);
        else {
          const float lim = __fmul_rn(alpha, dd);
          th = last_true([&](int S) { return __int2float_rn(S) < lim; }, lim);
        }
        th -= nrm;  // |th| <= 2^30 + 2^28: no overflow
        if (dd == 0.0f) atomicOr(&zmask[i >> 5], 1u << (i & 31));
      }
      ns[i] = th;   // folded threshold
      sn[i] = nrm;  // sorted norm (0 for IP and padding)
    }
    __syncthreads();
    // Re-prune lists start with the target's row, whose first nS entries are a
    // prune output: no entry of that prefix S culls a later one (same exact
    // distances, same test). Only pairs with an entry of the unverified tail U
    // need testing: U x S and U x U Gram tiles instead of the full triangle.
    uint32_t nS = 0;
    if (a.row_lists && a.spre && m2 == m) nS = min(cur.spre, m);
    const bool su = nS >= 16 && nS < m && nS <= P;
    if (su) {
      uint16_t* ipos = reinterpret_cast<uint16_t*>(tk);  // input index -> sorted position
      for (uint32_t r = tid; r < m2; r += NT) ipos[perm[r]] = static_cast<uint16_t>(r);
      __syncthreads();
      const uint32_t nu = m - nS;
      const uint32_t mu = (nu + 15) >> 4;             // U row tiles
      const uint32_t ncS = (nS + 15) >> 4, ncU = mu;  // S / U column tiles
      const uint32_t items = mu * (ncS + ncU);
      const int g = lane >> 2, tg = lane & 3;
      for (uint32_t it = warp; it < items; it += NT / 32) {
        const uint32_t ru = it / (ncS + ncU), cc = it - ru * (ncS + ncU);
        const bool isU = cc >= ncS;
        const uint32_t cb = isU ? cc - ncS : cc;
        const uint32_t cbase = isU ? nS : 0u, cend = isU ? m : nS;
        const uint32_t al = ru * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const uint32_t ia = nS + al < m ? nS + al : mc;
        const uint32_t bl = cbase + cb * 16 + (lane & 7) + (lane >> 4) * 8;
        const uint32_t ib = bl < cend ? bl : mc;
        const uint8_t* arow = X + size_t(ia) * xs + (lane >> 4) * 16;
        const uint8_t* brow = X + size_t(ib) * xs + ((lane >> 3) & 1) * 16;
        int acc0[4] = {0, 0, 0, 0}, acc1[4] = {0, 0, 0, 0};
        for (uint32_t kc = 0; kc < (kp >> 5); kc++) {
          uint32_t af[4], bf[4];
          ldsm_x4(af, arow + kc * 32);
          ldsm_x4(bf, brow + kc * 32);
          mma_i8<SIGNED>(acc0, af, bf[0], bf[1]);
          mma_i8<SIGNED>(acc1, af, bf[2], bf[3]);
        }
#pragma unroll
        for (int rr = 0; rr < 2; rr++) {
          const uint32_t ui = nS + ru * 16 + g + rr * 8;
          if (ui >= m) continue;
          const uint32_t pu = ipos[ui];
#pragma unroll
          for (int h = 0; h < 2; h++) {
#pragma unroll
            for (int e2 = 0; e2 < 2; e2++) {
              const uint32_t ci = cbase + cb * 16 + h * 8 + tg * 2 + e2;
              if (ci >= cend || ci == ui) continue;
              const uint32_t pc = ipos[ci];
              if (isU && pc < pu) continue;  // the (ci, ui) entry tests this pair
              const uint32_t x = pu < pc ? pu : pc, y = pu < pc ? pc : pu;  // x precedes y
              if ((zmask[x >> 5] >> (x & 31)) & 1u) continue;  // prune.cpp:32
              const int gram = h ? acc1[rr * 2 + e2] : acc0[rr * 2 + e2];
              const int gm = M == kL2 ? -2 * gram : -gram;
              const bool cull = RULE == 0 ? (sn[x] + gm <= ns[y]) : (sn[y] + gm <= ns[x]);
              if (cull) atomicOr(&cm[x * W + (y >> 5)], 1u << (y & 31));
            }
          }
        }
      }
    } else
    // all cull tests of the upper triangle (sorted positions), 16x16 tiles per warp
    {
      const uint32_t mt = mpad >> 4;
      const int g = lane >> 2, tg = lane & 3;
      // upper-triangle tiles in column-major order (it = cb (cb + 1) / 2 + rb),
      // warp w takes it = w, w + 4, ...; (cb, rb) advance incrementally
      uint32_t cb = 0, rb = static_cast<uint32_t>(warp);
      while (rb > cb) {
        rb -= cb + 1;
        cb++;
      }
      for (; cb < mt; ) {
        const uint32_t r0 = rb * 16, n0 = cb * 16;
        const uint32_t ar = r0 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const uint32_t br = n0 + (lane & 7) + (lane >> 4) * 8;
        const uint8_t* arow = X + size_t(ar < m2 ? perm[ar] : mc) * xs + (lane >> 4) * 16;
        const uint8_t* brow = X + size_t(br < m2 ? perm[br] : mc) * xs + ((lane >> 3) & 1) * 16;
        int acc0[4] = {0, 0, 0, 0}, acc1[4] = {0, 0, 0, 0};
        for (uint32_t kc = 0; kc < (kp >> 5); kc++) {
          uint32_t af[4], bf[4];
          ldsm_x4(af, arow + kc * 32);
          ldsm_x4(bf, brow + kc * 32);
          mma_i8<SIGNED>(acc0, af, bf[0], bf[1]);
          mma_i8<SIGNED>(acc1, af, bf[2], bf[3]);
        }
        // this lane's two rows and four columns of the tile
        // rule 0: cull iff |x_i|^2 - 2 g <= T_j - |x_j|^2 (column threshold)
        // rule 1: cull iff |x_j|^2 - 2 g <= V_i - |x_i|^2 (row threshold)
        // (IP: norms 0, -g in place of -2 g)
        uint32_t vmask[2];  // columns (bit = tile column) this row may cull
        int rv[2];          // rule 0: |x_i|^2 ; rule 1: row threshold
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const uint32_t row = r0 + g + h * 8;
          // prune.cpp:32: a zero-distance pick culls nothing; only columns
          // right of the row and inside the list
          const bool live = row < m2 && ((zmask[row >> 5] >> (row & 31)) & 1u) == 0;
          const uint32_t right = row < n0 ? 0xFFFFu : (row - n0 >= 15 ? 0u : (0xFFFFu << (row - n0 + 1)) & 0xFFFFu);
          const uint32_t inside = m2 >= n0 + 16 ? 0xFFFFu : (m2 <= n0 ? 0u : (1u << (m2 - n0)) - 1u);
          vmask[h] = live ? (right & inside) : 0u;
          rv[h] = RULE == 0 ? sn[row] : ns[row];
        }
        uint32_t bits[2] = {0u, 0u};
#pragma unroll
        for (int h = 0; h < 2; h++) {
#pragma unroll
          for (int e2 = 0; e2 < 2; e2++) {
            const uint32_t ccol = h * 8 + tg * 2 + e2;
            const uint32_t col = n0 + ccol;
            // rule 0: column threshold; rule 1: column norm
            const int cv = RULE == 0 ? ns[col] : sn[col];
#pragma unroll
            for (int rr = 0; rr < 2; rr++) {
              const int gram = h ? acc1[rr * 2 + e2] : acc0[rr * 2 + e2];
              const int gm = M == kL2 ? -2 * gram : -gram;
              const bool cull = RULE == 0 ? (rv[rr] + gm <= cv) : (cv + gm <= rv[rr]);
              if (cull) bits[rr] |= 1u << ccol;
            }
          }
        }
        uint32_t bits_lo = bits[0] & vmask[0], bits_hi = bits[1] & vmask[1];
        rb += NT / 32;
        while (rb > cb) {
          rb -= cb + 1;
          cb++;
        }
        bits_lo |= __shfl_xor_sync(FULL, bits_lo, 1);
        bits_lo |= __shfl_xor_sync(FULL, bits_lo, 2);
        bits_hi |= __shfl_xor_sync(FULL, bits_hi, 1);
        bits_hi |= __shfl_xor_sync(FULL, bits_hi, 2);
        if (tg == 0) {
          const uint32_t sh = n0 & 31;
          if (bits_lo) atomicOr(&cm[(r0 + g) * W + (n0 >> 5)], bits_lo << sh);
          if (bits_hi) atomicOr(&cm[(r0 + g + 8) * W + (n0 >> 5)], bits_hi << sh);
        }
      }
    }
    __syncthreads();
    // hand off: [m2][sorted ids][zero mask][cull rows]
    if (tid == 0) out[0] = m2;
    for (uint32_t i = tid; i < m2; i += NT) out[4 + i] = key_id(sk[i]);
    for (uint32_t i = tid; i < W; i += NT) out[4 + mc + i] = i < mw ? zmask[i] : 0u;
    uint4* dst = reinterpret_cast<uint4*>(out + 4 + mc + W);
    const uint4* srcm = reinterpret_cast<const uint4*>(cm);
    for (uint32_t i = tid; i < m2 * (W / 4); i += NT) dst[i] = srcm[i];
    if (tid == 0 && a.stats) {
      atomicAdd(stat_slot(a.stats) + kStPruneLists, 1ull);
      atomicAdd(stat_slot(a.stats) + kStPruneCands, static_cast<unsigned long long>(m));
      // pair tests evaluated on the tensor cores
      atomicAdd(stat_slot(a.stats) + kStPruneEvals, static_cast<unsigned long long>(m2) * (m2 - (m2 > 0)) / 2);
    }
  }
}

// Stage 2: the greedy walk, one warp per list. The list's cull rows are staged
// in shared memory with coalesced loads; every lane carries the whole culled
// set in W registers and the next row is read before the current decision, so
// the chain per candidate is a bit test and an OR (prune.cpp:25-43).
constexpr int kWalkWarps = 4;
template <int W>
__global__ void __launch_bounds__(kWalkWarps * 32)
    prune_walk_kernel(const PruneArgs a, const MmaLayout ly, const uint32_t* hand, uint32_t l0, uint32_t lcount) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint4* srows = reinterpret_cast<uint4*>(smem) + size_t(wib) * ly.mc * (W / 4);
  const uint32_t rel = blockIdx.x * kWalkWarps + wib;
  if (rel >= lcount) return;
  const uint32_t li = l0 + rel;
  const uint32_t l = a.list_index ? a.list_index[li] : li;
  const uint32_t m = a.lengths[l];
  if (m < a.mmin || m > a.mcap) return;
  const uint32_t p = a.points[l];
  const uint32_t R = a.R;
  uint32_t* orow = a.out_rows ? a.out_rows + uint64_t(l) * R : a.out_adj + uint64_t(p - a.out_base) * R;
  const uint32_t* in = hand + size_t(rel) * ly.stride;
  const uint32_t m2 = in[0];
  const uint32_t* ids = in + 4;
  const uint32_t* zm = ids + ly.mc;
  const uint4* rows = reinterpret_cast<const uint4*>(zm + W);
  for (uint32_t i = lane; i < m2 * (W / 4); i += 32) srows[i] = rows[i];
  uint32_t culled[W], z[W];
#pragma unroll
  for (int w = 0; w < W; w++) {
    culled[w] = 0u;
    z[w] = zm[w];
  }
  __syncwarp();
  uint32_t nsel = 0;
  uint4 nxt[W / 4];
#pragma unroll
  for (int q = 0; q < W / 4; q++) nxt[q] = srows[q];
#pragma unroll
  for (int w = 0; w < W; w++) {
    if (32u * w >= m2 || nsel == R) break;
    for (uint32_t b = 0; b < 32; b++) {
      const uint32_t i = 32u * w + b;
      if (i >= m2) break;
      uint4 cur[W / 4];
#pragma unroll
      for (int q = 0; q < W / 4; q++) cur[q] = nxt[q];
      if (i + 1 < m2) {
#pragma unroll
        for (int q = 0; q < W / 4; q++) nxt[q] = srows[size_t(i + 1) * (W / 4) + q];
      }
      if ((culled[w] >> b) & 1u) continue;
      if (lane == 0) orow[nsel] = ids[i];
      nsel++;
      if (nsel == R) break;
      if ((z[w] >> b) & 1u) continue;
#pragma unroll
      for (int q = 0; q < W / 4; q++) {
        culled[4 * q + 0] |= cur[q].x;
        culled[4 * q + 1] |= cur[q].y;
        culled[4 * q + 2] |= cur[q].z;
        culled[4 * q + 3] |= cur[q].w;
      }
    }
  }
  for (uint32_t i = nsel + lane; i < R; i += 32) orow[i] = kNone;
  if (lane == 0 && a.n_out) a.n_out[l] = nsel;
  // a prune output: no entry culls a later one (exact int distances), so a
  // later re-prune of this row + appended sources may skip those pairs
  if (lane == 0 && a.spre && !a.out_rows) a.spre[p - a.out_base] = static_cast<uint8_t>(nsel < 255 ? nsel : 255);
}

// ---- length binning --------------------------------------------------------
// Splits the lists of a launch into kBins length bins (bounds[b-1], bounds[b]]
// so each bin's prune launch covers only its own lists.
__global__ void bin_lists_kernel(const PruneArgs a, const uint32_t* bounds, int nb, uint32_t* counts,
                                 uint32_t* lists, uint32_t cap) {
  const uint32_t li = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = li < a.count;
  const uint32_t l = valid ? (a.list_index ? a.list_index[li] : li) : 0u;
  const uint32_t m = valid ? a.lengths[l] : 0u;
  int b = nb + 2;  // longer than every bound
  if (valid)
    for (int i = 0; i < nb; i++)
      if (m <= bounds[i]) {
        b = i;
        break;
      }
  if (valid && a.small_u && a.row_lists && a.spre) {  // the warp re-prune's classes (bins nb: few entries, nb + 1)
    const uint32_t S = min(static_cast<uint32_t>(a.spre[a.points[l] - a.out_base]), m);
    if (S <= 64 && m - S <= a.small_u) b = (a.small_u2 && m - S <= a.small_u2) ? nb : nb + 1;
  }
  for (int i = 0; i <= nb + 1; i++) {  // warp-aggregated append per bin
    const uint32_t mask = __ballot_sync(0xFFFFFFFFu, b == i);
    if (!mask) continue;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(counts + i, __popc(mask));
    base = __shfl_sync(0xFFFFFFFFu, base, leader);
    if (b == i) lists[size_t(i) * cap + base + __popc(mask & ((1u << lane) - 1u))] = l;
  }
}

cudaError_t launch_bin_lists(const PruneArgs& a, const uint32_t* d_bounds, int nb, uint32_t* d_counts,
                             uint32_t* d_lists, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(d_counts, 0, sizeof(uint32_t) * (nb + 2), s);  // + the warp re-prune's two classes
  if (e != cudaSuccess || a.count == 0) return e;
  bin_lists_kernel<<<(a.count + 255) / 256, 256, 0, s>>>(a, d_bounds, nb, d_counts, d_lists, a.count);
  return cudaGetLastError();
}

// ---- back-edge re-prunes of a row plus a few sources: one warp per list -------
// apply_back_edges (src/builder_common.cpp:109-140) re-prunes a target t whose
// merged list (its row ++ new sources) outgrew R. The row's first spre
// entries are a previous prune's output under the same alpha and rule:
// sorted by (d(t, .), id) and mutually non-culling (no earlier entry of it
// culls a later one). With u = m - spre <= kSmallU other entries, the greedy
// of src/prune.cpp:25-43 only needs the tests that involve those u entries:
//   * u_k is culled iff a selected entry before it (an S entry, or an earlier
//     selected u) culls it;
//   * an S entry is culled iff a selected u before it culls it;
// and the selection stops at R. So one warp computes d(t, x) for the m rows
// and d(u_i, s) for the u x spre pairs — every S row gathered once, its norm,
// its dot products with t and the u rows reduced across the row's lanes — and
// walks the u entries in key order. No shared memory, no block barrier, no
// tensor-core tile (the prep kernel's Gram tile was 3.8% tensor-pipe busy on
// these lists, barrier stalls 24%: profiles/r01e_prune_prep_reprune_c1.txt).
constexpr int kSmallU = 4;
constexpr int kSmallU2 = 2;  // the lists with at most this many get the smaller instance

template <int E>
__device__ __forceinline__ int dot_chunk(const uint4& a, const uint4& b, int acc) {
  if (E == kI8) {
    acc = __dp4a(static_cast<int>(a.x), static_cast<int>(b.x), acc);
    acc = __dp4a(static_cast<int>(a.y), static_cast<int>(b.y), acc);
    acc = __dp4a(static_cast<int>(a.z), static_cast<int>(b.z), acc);
    return __dp4a(static_cast<int>(a.w), static_cast<int>(b.w), acc);
  }
  uint32_t u = static_cast<uint32_t>(acc);
  u = __dp4a(a.x, b.x, u);
  u = __dp4a(a.y, b.y, u);
  u = __dp4a(a.z, b.z, u);
  return static_cast<int>(__dp4a(a.w, b.w, u));
}

// The exact pair distance from norms and the dot product (integer kinds):
// |x|^2 + |y|^2 - 2 x.y is the int32 sum the reference accumulates
// (src/metric.cpp:38-59); IP is -x.y.
template <int M>
__device__ __forceinline__ float pair_dist(int nx, int ny, int dot) {
  if (M == kIP) return -__int2float_rn(dot);
  return __int2float_rn(nx + ny - 2 * dot);
}

// cull(i -> j) of src/prune.cpp:36-39 (i selected, j later; di = d(t, i),
// dj = d(t, j), via = d(i, j)); a zero-distance pick culls nothing (:32).
__device__ __forceinline__ bool cull_test(int rule, float alpha, float di, float dj, float via) {
  if (di == 0.0f) return false;
  return rule == 0 ? __fmul_rn(alpha, via) <= dj : via < __fmul_rn(alpha, di);
}

// KU: the most non-prefix entries a list of this instance has (2 or KU: the
// smaller instance holds fewer rows and sums in registers)
#ifndef GANN_RS_MINB4
#define GANN_RS_MINB4 6  // resident CTAs the KU = 4 instance's registers are budgeted for (6: 80 registers, 56 B spilled; measured: 4 CTAs at 128 registers re-prune phase 681 ms, 5: 684, 6: 667)
#endif
#ifndef GANN_RS_MINB2
#define GANN_RS_MINB2 8  // ... the KU = 2 instance's (8: 64 registers; 7 CTAs at 72: 681 ms, 8: 661)
#endif
template <int E, int M, int LPR, int CPL, int KU>
__global__ void __launch_bounds__(128, KU > 2 ? GANN_RS_MINB4 : GANN_RS_MINB2) reprune_small_kernel(const PruneArgs a) {
  constexpr int RPP = 32 / LPR;  // rows per warp pass (one per lane group)
  const int lane = threadIdx.x & 31;
  const int sub = lane & (LPR - 1), grp = lane / LPR;
  const uint32_t nch = static_cast<uint32_t>(a.stride >> 4);
  const uint32_t R = a.R;
  const float alpha = a.alpha;
  const uint32_t FULL = 0xFFFFFFFFu;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t li = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; li < a.count; li += warps) {
    const uint32_t l = a.list_index ? a.list_index[li] : li;
    const uint32_t m = a.lengths[l];
    const uint32_t p = a.points[l];
    const uint64_t beg = a.begins ? a.begins[l] : uint64_t(l) * a.fixed_stride;
    const uint32_t S = min(static_cast<uint32_t>(a.spre[p - a.out_base]), m);
    const uint32_t nu = m - S;  // <= KU (binned by the host), S <= 64
    // ids: S entries two per lane (index lane, lane + 32); the u entries in every lane
    const uint32_t s0 = lane < S ? __ldg(a.cand_ids + beg + lane) : kNone;
    const uint32_t s1 = lane + 32 < S ? __ldg(a.cand_ids + beg + 32 + lane) : kNone;
    uint32_t uid[KU];
#pragma unroll
    for (int i = 0; i < KU; i++) uid[i] = i < static_cast<int>(nu) ? __ldg(a.cand_ids + beg + S + i) : kNone;
    // the lane's chunks of t's row and of the u rows, their norms and d(t, u_i)
    uint4 qt[CPL], qu[KU][CPL];
    bool chv[CPL];
#pragma unroll
    for (int c = 0; c < CPL; c++) {
      const uint32_t ch = sub + c * LPR;
      chv[c] = ch < nch;
      qt[c] = chv[c] ? __ldg(reinterpret_cast<const uint4*>(a.data + uint64_t(p) * a.stride) + ch) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int i = 0; i < KU; i++)
        qu[i][c] = (chv[c] && uid[i] != kNone)
                       ? __ldg(reinterpret_cast<const uint4*>(a.data + uint64_t(uid[i]) * a.stride) + ch)
                       : make_uint4(0, 0, 0, 0);
    }
    int nt = 0, nuv[KU], dtu[KU], duu[KU][KU];
#pragma unroll
    for (int c = 0; c < CPL; c++) nt = dot_chunk<E>(qt[c], qt[c], nt);
    nt = group_sum<LPR>(nt);
#pragma unroll
    for (int i = 0; i < KU; i++) {
      int n = 0, d = 0;
#pragma unroll
      for (int c = 0; c < CPL; c++) {
        n = dot_chunk<E>(qu[i][c], qu[i][c], n);
        d = dot_chunk<E>(qt[c], qu[i][c], d);
      }
      nuv[i] = group_sum<LPR>(n);
      dtu[i] = group_sum<LPR>(d);
#pragma unroll
      for (int j = 0; j < KU; j++) {
        int x = 0;
        if (j > i) {
#pragma unroll
          for (int c = 0; c < CPL; c++) x = dot_chunk<E>(qu[i][c], qu[j][c], x);
          x = group_sum<LPR>(x);
        }
        duu[i][j] = x;
      }
    }
    float du_t[KU];  // d(t, u_i)
#pragma unroll
    for (int i = 0; i < KU; i++) du_t[i] = pair_dist<M>(nt, nuv[i], dtu[i]);
    // S rows: lane group g takes rows g, g + RPP, ...; per row the norm and the
    // dots with t and the u rows, reduced over the group's lanes; lane
    // (row & 31) keeps the row's values (rows r and r + 32 of the same lane)
    float dts[2] = {0.0f, 0.0f};              // d(t, s)
    float dus[2][KU];                     // d(u_i, s)
#pragma unroll
    for (int h = 0; h < 2; h++)
#pragma unroll
      for (int i = 0; i < KU; i++) dus[h][i] = 0.0f;
    // UU rows per lane group in flight; the sums reduced with the transposed
    // butterfly (lane sub of group g ends with row g*UU + (sub mod UU))
    constexpr int UU = LPR >= 4 ? 4 : LPR;
    constexpr int PASS = RPP * UU;  // rows per warp pass (divides 32 for LPR >= 4)
    for (uint32_t r0 = 0; r0 < S; r0 += PASS) {
      uint4 x[UU][CPL];
#pragma unroll
      for (int u = 0; u < UU; u++) {
        const uint32_t r = r0 + grp * UU + u;
        const uint32_t id = __shfl_sync(FULL, r0 < 32 ? s0 : s1, r & 31);
#pragma unroll
        for (int c = 0; c < CPL; c++)
          x[u][c] = (r < S && chv[c]) ? __ldg(reinterpret_cast<const uint4*>(a.data + uint64_t(id) * a.stride) + sub + c * LPR)
                                      : make_uint4(0, 0, 0, 0);
      }
      int ns[UU], dt[UU], du[KU][UU];
#pragma unroll
      for (int u = 0; u < UU; u++) {
        ns[u] = 0;
        dt[u] = 0;
#pragma unroll
        for (int i = 0; i < KU; i++) du[i][u] = 0;
#pragma unroll
        for (int c = 0; c < CPL; c++) {
          ns[u] = dot_chunk<E>(x[u][c], x[u][c], ns[u]);
          dt[u] = dot_chunk<E>(qt[c], x[u][c], dt[u]);
#pragma unroll
          for (int i = 0; i < KU; i++) du[i][u] = dot_chunk<E>(qu[i][c], x[u][c], du[i][u]);
        }
      }
      const int ns_g = transpose_reduce<LPR, UU>(ns, sub);
      const int dt_g = transpose_reduce<LPR, UU>(dt, sub);
      int du_g[KU];
#pragma unroll
      for (int i = 0; i < KU; i++) du_g[i] = transpose_reduce<LPR, UU>(du[i], sub);
      // lane (row & 31) takes its row's sums (row r0 + g*UU + u sits in lane g*LPR + u)
      const int j = lane - static_cast<int>(r0 & 31u);
      const bool mine = j >= 0 && j < PASS && r0 + j < S;
      const int src = mine ? (j / UU) * LPR + (j % UU) : 0;
      const int ns_r = __shfl_sync(FULL, ns_g, src), dt_r = __shfl_sync(FULL, dt_g, src);
      int du_r[KU];
#pragma unroll
      for (int i = 0; i < KU; i++) du_r[i] = __shfl_sync(FULL, du_g[i], src);
      if (mine) {  // (static indices: the arrays stay in registers)
        if (r0 >= 32) {
          dts[1] = pair_dist<M>(nt, ns_r, dt_r);
#pragma unroll
          for (int i = 0; i < KU; i++) dus[1][i] = pair_dist<M>(nuv[i], ns_r, du_r[i]);
        } else {
          dts[0] = pair_dist<M>(nt, ns_r, dt_r);
#pragma unroll
          for (int i = 0; i < KU; i++) dus[0][i] = pair_dist<M>(nuv[i], ns_r, du_r[i]);
        }
      }
    }
    // keys; S must be ascending (a prune's output): else leave the list to
    // the general kernel (flagged through too_long; never seen in the tests)
    const uint64_t ks0 = lane < S ? make_key(dts[0], s0) : kMaxKey;
    const uint64_t ks1 = lane + 32 < S ? make_key(dts[1], s1) : kMaxKey;
    uint64_t ku[KU];
#pragma unroll
    for (int i = 0; i < KU; i++) ku[i] = uid[i] != kNone && uid[i] != p ? make_key(du_t[i], uid[i]) : kMaxKey;
    {
      const uint64_t nx = __shfl_down_sync(FULL, ks0, 1);
      const uint64_t n32 = __shfl_sync(FULL, ks1, 0);
      const uint64_t nx1 = __shfl_down_sync(FULL, ks1, 1);
      const bool bad = (lane + 1 < S && (lane < 31 ? nx : n32) <= ks0) || (lane + 33 < S && nx1 <= ks1);
      if (__any_sync(FULL, bad)) {
        if (lane == 0) atomicAdd(a.too_long, 1u);
        continue;
      }
    }
    // u entries in key order; each one's count of S keys below it
    int ord[KU];
    uint32_t below[KU];
#pragma unroll
    for (int i = 0; i < KU; i++) {
      int r = 0;
#pragma unroll
      for (int j = 0; j < KU; j++) r += ku[j] < ku[i] ? 1 : 0;
      ord[i] = r;
      below[i] = __popc(__ballot_sync(FULL, ks0 < ku[i])) + __popc(__ballot_sync(FULL, ks1 < ku[i]));
    }
    // the walk: u entries in key order; S entries culled only by selected u's
    bool cs0 = lane >= S, cs1 = lane + 32 >= S;  // culled (or absent)
    bool selu[KU];
#pragma unroll
    for (int i = 0; i < KU; i++) selu[i] = false;
    bool full = false;
#pragma unroll
    for (int o = 0; o < KU; o++) {
#pragma unroll
      for (int k = 0; k < KU; k++) {  // k: the u entry of rank o (warp-uniform test)
        if (ord[k] != o || ku[k] == kMaxKey || full) continue;
        const uint32_t bk = below[k];
        // selected S entries before it (S index < bk), and whether one culls it
        const bool e0 = !cs0 && static_cast<uint32_t>(lane) < bk;
        const bool e1 = !cs1 && static_cast<uint32_t>(lane) + 32 < bk;
        bool c = (e0 && cull_test(a.rule, alpha, dts[0], du_t[k], dus[0][k])) ||
                 (e1 && cull_test(a.rule, alpha, dts[1], du_t[k], dus[1][k]));
        uint32_t before = __popc(__ballot_sync(FULL, e0)) + __popc(__ballot_sync(FULL, e1));
        c = __any_sync(FULL, c);
#pragma unroll
        for (int j = 0; j < KU; j++) {
          if (j == k || !selu[j] || ord[j] >= o) continue;
          before++;
          const int dij = j < k ? duu[j][k] : duu[k][j];
          c = c || cull_test(a.rule, alpha, du_t[j], du_t[k], pair_dist<M>(nuv[j], nuv[k], dij));
        }
        if (before >= R) {
          full = true;
          continue;
        }
        if (c) continue;
        selu[k] = true;
        // it culls the S entries after it
        if (du_t[k] != 0.0f) {
          if (!cs0 && static_cast<uint32_t>(lane) >= bk && cull_test(a.rule, alpha, du_t[k], dts[0], dus[0][k]))
            cs0 = true;
          if (!cs1 && static_cast<uint32_t>(lane) + 32 >= bk && cull_test(a.rule, alpha, du_t[k], dts[1], dus[1][k]))
            cs1 = true;
        }
      }
    }
    // output: selected entries in key order, the first R of them
    uint32_t* orow = a.out_rows ? a.out_rows + uint64_t(l) * R : a.out_adj + uint64_t(p - a.out_base) * R;
    const uint32_t b0 = __ballot_sync(FULL, !cs0), b1 = __ballot_sync(FULL, !cs1);
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t nsel = __popc(b0) + __popc(b1);
#pragma unroll
    for (int i = 0; i < KU; i++) nsel += selu[i] ? 1u : 0u;
    nsel = min(nsel, R);
    auto selu_before = [&](uint32_t sidx) {  // selected u entries sorting before S index sidx
      uint32_t n = 0;
#pragma unroll
      for (int i = 0; i < KU; i++) n += (selu[i] && below[i] <= sidx) ? 1u : 0u;
      return n;
    };
    GANN_CHECK(S <= 64 && nu <= KU);
    if (!cs0) {
      const uint32_t oi = __popc(b0 & lt) + selu_before(lane);
      if (oi < R) orow[oi] = s0;
    }
    if (!cs1) {
      const uint32_t oi = __popc(b0) + __popc(b1 & lt) + selu_before(lane + 32);
      if (oi < R) orow[oi] = s1;
    }
    if (lane == 0) {
      auto lowmask = [](uint32_t k) { return k >= 32 ? 0xFFFFFFFFu : (1u << k) - 1u; };
#pragma unroll
      for (int i = 0; i < KU; i++) {
        if (!selu[i]) continue;
        uint32_t oi = 0;  // selected S below it + selected u before it
        oi += __popc(b0 & lowmask(below[i]));
        oi += below[i] > 32 ? __popc(b1 & lowmask(below[i] - 32)) : 0u;
#pragma unroll
        for (int j = 0; j < KU; j++) oi += (selu[j] && ord[j] < ord[i]) ? 1u : 0u;
        if (oi < R) orow[oi] = uid[i];
      }
      if (a.stats) {
        atomicAdd(stat_slot(a.stats) + kStPruneLists, 1ull);
        atomicAdd(stat_slot(a.stats) + kStPruneCands, static_cast<unsigned long long>(m));
      }
    }
    for (uint32_t i = nsel + lane; i < R; i += 32) orow[i] = kNone;
    if (lane == 0) {
      if (a.n_out) a.n_out[l] = nsel;
      if (a.spre && !a.out_rows) a.spre[p - a.out_base] = static_cast<uint8_t>(nsel < 255 ? nsel : 255);
    }
  }
}

// ---- long lists: chunked prune ------------------------------------------------
// Exact restatement of the same greedy for lists of any length (back-edge
// hubs). The candidates are consumed in key order, C at a time: a radix select
// over the (dist, id) keys finds the C smallest keys above the previous
// chunk's last key; those are sorted in shared memory, first culled by every
// non-zero-distance selection of the earlier chunks (an element is culled iff
// some earlier selection's test fires on it — the order of the tests does not
// matter), then walked greedily as above. Most hubs finish inside the first
// chunk because R selections are reached long before the list ends.
constexpr uint32_t kChunk = 512;

size_t prune_chunked_smem(uint32_t R) {
  size_t b = size_t(kChunk) * 8 + 2 * size_t(kChunk) * 2 + kChunk + size_t(R) * 8 + 256 * 4;
  return (b + 15) & ~size_t(15);
}

template <int E, int M, int LPR, int CPL, int NT>
__global__ void __launch_bounds__(NT) prune_chunked_kernel(const PruneArgs a) {
  using Op = DistOp<E, M>;
  constexpr int GROUPS = NT / LPR;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t warp_tot[NT / 32];
  __shared__ uint32_t sh_cnt;
  __shared__ uint64_t sh_prefix;
  __shared__ uint32_t sh_want;
  __shared__ unsigned long long sh_evals;
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  uint16_t* alA = reinterpret_cast<uint16_t*>(keys + kChunk);
  uint16_t* alB = alA + kChunk;
  uint8_t* kf = reinterpret_cast<uint8_t*>(alB + kChunk);
  uint32_t* sel = reinterpret_cast<uint32_t*>(kf + kChunk);
  float* seld = reinterpret_cast<float*>(sel + a.R);
  uint32_t* hist = reinterpret_cast<uint32_t*>(seld + a.R);
  const int tid = threadIdx.x;
  const int sub = tid & (LPR - 1);
  const int grp = tid / LPR;
  const uint32_t nch = static_cast<uint32_t>(a.stride >> 4);
  const uint32_t R = a.R;

  for (uint32_t li = blockIdx.x; li < a.count; li += gridDim.x) {
    const uint32_t l = a.list_index ? a.list_index[li] : li;
    const uint32_t p = a.points[l];
    const uint64_t beg = a.begins ? a.begins[l] : uint64_t(l) * a.fixed_stride;
    const uint64_t m = a.lengths[l];
    uint32_t* orow = a.out_rows ? a.out_rows + uint64_t(l) * R : a.out_adj + uint64_t(p - a.out_base) * R;
    if (m < a.mmin) continue;
    if (m > a.mcap) {  // only mcap entries exist (a walk that outgrew its buffer): re-run by the caller
      if (tid == 0 && !a.skip_long) atomicAdd(a.too_long, 1u);
      continue;
    }
    auto key_at = [&](uint64_t i) -> uint64_t {
      const uint32_t id = a.cand_ids[beg + i];
      return id == p ? kMaxKey : make_key(a.cand_dists[beg + i], id);
    };
    uint64_t lo_key = 0;        // keys <= lo_key are done
    bool first = true;
    uint32_t nsel = 0;
    uint64_t evals = 0;
    if (tid == 0) sh_evals = 0;
    while (nsel < R) {
      // how many keys remain above lo_key?
      if (tid == 0) sh_cnt = 0;
      __syncthreads();
      uint32_t local = 0;
      for (uint64_t i = tid; i < m; i += NT) {
        const uint64_t k = key_at(i);
        local += (k != kMaxKey && (first || k > lo_key)) ? 1u : 0u;
      }
      atomicAdd(&sh_cnt, local);
      __syncthreads();
      const uint32_t rem = sh_cnt;
      if (rem == 0) break;
      uint64_t hi_key = kMaxKey - 1;
      if (rem > kChunk) {  // radix select of the kChunk-th smallest key above lo_key
        if (tid == 0) {
          sh_prefix = 0;
          sh_want = kChunk;
        }
        for (int shift = 56; shift >= 0; shift -= 8) {
          for (int b = tid; b < 256; b += NT) hist[b] = 0;
          __syncthreads();
          const uint64_t prefix = sh_prefix;
          const uint64_t hmask = shift == 56 ? 0ull : (~0ull << (shift + 8));
          for (uint64_t i = tid; i < m; i += NT) {
            const uint64_t k = key_at(i);
            if (k != kMaxKey && (first || k > lo_key) && (k & hmask) == prefix)
              atomicAdd(&hist[(k >> shift) & 0xFF], 1u);
          }
          __syncthreads();
          if (tid == 0) {
            uint32_t want = sh_want, acc = 0;
            int b = 0;
            for (; b < 256; b++) {
              if (acc + hist[b] >= want) break;
              acc += hist[b];
            }
            sh_want = want - acc;
            sh_prefix = prefix | (uint64_t(b) << shift);
          }
          __syncthreads();
        }
        hi_key = sh_prefix;
      }
      // gather the chunk (lo_key, hi_key] and sort it; every thread has read
      // rem = sh_cnt before it is reset (without this barrier a warp could
      // read the reset count when rem <= kChunk skips the radix select's)
      __syncthreads();
      if (tid == 0) sh_cnt = 0;
      __syncthreads();
      for (uint64_t i = tid; i < m; i += NT) {
        const uint64_t k = key_at(i);
        if (k != kMaxKey && (first || k > lo_key) && k <= hi_key) {
          const uint32_t pos = atomicAdd(&sh_cnt, 1u);
          if (pos < kChunk) keys[pos] = k;  // only exact duplicate keys can overflow
        }
      }
      __syncthreads();
      const uint32_t c = min(sh_cnt, kChunk);
      uint32_t Mp = 32;
      while (Mp < c) Mp <<= 1;
      for (uint32_t i = c + tid; i < Mp; i += NT) keys[i] = kMaxKey;
      __syncthreads();
      for (uint32_t k = 2; k <= Mp; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
          for (uint32_t i = tid; i < Mp; i += NT) {
            const uint32_t ixj = i ^ j;
            if (ixj > i) {
              const uint64_t x = keys[i], y = keys[ixj];
              if ((x > y) == ((i & k) == 0)) {
                keys[i] = y;
                keys[ixj] = x;
              }
            }
          }
          __syncthreads();
        }
      }
      // cull the chunk by the earlier chunks' selections
      for (uint32_t b0 = 0; b0 < c; b0 += GROUPS) {
        const uint32_t t = b0 + grp;
        bool culled = false;
        if (nsel > 0) {
          uint4 x[CPL];
          const uint32_t id = t < c ? key_id(keys[t]) : 0u;
          const float dj = t < c ? key_dist(keys[t]) : 0.0f;
          const uint8_t* rp = a.data + uint64_t(id) * a.stride;
#pragma unroll
          for (int cc = 0; cc < CPL; cc++) {
            const uint32_t ch = sub + cc * LPR;
            x[cc] = (t < c && ch < nch) ? __ldg(reinterpret_cast<const uint4*>(rp) + ch) : make_uint4(0, 0, 0, 0);
          }
          for (uint32_t s2 = 0; s2 < nsel; s2++) {  // warp-uniform trip count (shuffles inside)
            if (__all_sync(0xFFFFFFFFu, culled)) break;
            const float sd = seld[s2];
            if (sd == 0.0f) continue;
            const uint8_t* sp = a.data + uint64_t(sel[s2]) * a.stride;
            typename Op::acc_t acc = Op::zero();
#pragma unroll
            for (int cc = 0; cc < CPL; cc++) {
              const uint32_t ch = sub + cc * LPR;
              const uint4 y = ch < nch ? __ldg(reinterpret_cast<const uint4*>(sp) + ch) : make_uint4(0, 0, 0, 0);
              acc = Op::chunk(y, x[cc], acc);
            }
            acc = group_sum<LPR>(acc);
            const float via = Op::finish(acc);
            if (!culled && sub == 0 && t < c) atomicAdd(&sh_evals, 1ull);
            culled = culled || (a.rule == 0 ? (__fmul_rn(a.alpha, via) <= dj) : (via < __fmul_rn(a.alpha, sd)));
          }
        }
        if (sub == 0 && t < c) {
          kf[t] = culled ? 0 : 1;
          alB[t] = static_cast<uint16_t>(t);
        }
      }
      __syncthreads();
      uint32_t nalive = cta_compact<NT>(alB, kf, c, alA, warp_tot);
      __syncthreads();
      uint16_t* alive = alA;
      while (nsel < R && nalive > 0) {
        const uint64_t sk = keys[alive[0]];
        if (tid == 0) {
          sel[nsel] = key_id(sk);
          seld[nsel] = key_dist(sk);
        }
        nsel++;
        if (nsel == R) break;
        if (key_dist(sk) == 0.0f) {
          alive++;
          nalive--;
          continue;
        }
        const uint32_t sid = key_id(sk);
        const float sdist = key_dist(sk);
        uint4 sr[CPL];
        const uint8_t* srow = a.data + uint64_t(sid) * a.stride;
#pragma unroll
        for (int cc = 0; cc < CPL; cc++) {
          const uint32_t ch = sub + cc * LPR;
          sr[cc] = ch < nch ? __ldg(reinterpret_cast<const uint4*>(srow) + ch) : make_uint4(0, 0, 0, 0);
        }
        const uint32_t rest = nalive - 1;
        evals += rest;
        for (uint32_t b0 = 0; b0 < rest; b0 += GROUPS) {
          const uint32_t t = b0 + grp;
          const uint32_t ix = t < rest ? alive[1 + t] : 0u;
          const uint32_t id = t < rest ? key_id(keys[ix]) : 0u;
          const uint8_t* rp = a.data + uint64_t(id) * a.stride;
          typename Op::acc_t acc = Op::zero();
#pragma unroll
          for (int cc = 0; cc < CPL; cc++) {
            const uint32_t ch = sub + cc * LPR;
            const uint4 x = (t < rest && ch < nch) ? __ldg(reinterpret_cast<const uint4*>(rp) + ch)
                                                   : make_uint4(0, 0, 0, 0);
            acc = Op::chunk(sr[cc], x, acc);
          }
          acc = group_sum<LPR>(acc);
          if (sub == 0 && t < rest) {
            const float via = Op::finish(acc);
            const float dj = key_dist(keys[ix]);
            const bool drop = a.rule == 0 ? (__fmul_rn(a.alpha, via) <= dj) : (via < __fmul_rn(a.alpha, sdist));
            kf[t] = drop ? 0 : 1;
          }
        }
        __syncthreads();
        uint16_t* dst = (alive >= alA && alive < alA + kChunk) ? alB : alA;
        nalive = cta_compact<NT>(alive + 1, kf, rest, dst, warp_tot);
        alive = dst;
        __syncthreads();
      }
      __syncthreads();
      if (rem <= kChunk) break;  // that was the last chunk
      lo_key = hi_key;
      first = false;
    }
    __syncthreads();
    for (uint32_t i = tid; i < R; i += NT) orow[i] = i < nsel ? sel[i] : kNone;
    if (tid == 0) {
      if (a.n_out) a.n_out[l] = nsel;
      if (a.spre && !a.out_rows) a.spre[p - a.out_base] = static_cast<uint8_t>(nsel < 255 ? nsel : 255);
      if (a.stats) {
        atomicAdd(stat_slot(a.stats) + kStPruneLists, 1ull);
        atomicAdd(stat_slot(a.stats) + kStPruneCands, static_cast<unsigned long long>(m));
        atomicAdd(stat_slot(a.stats) + kStPruneEvals, static_cast<unsigned long long>(evals) + sh_evals);
      }
    }
    __syncthreads();
  }
}

uint32_t reprune_small_max_u() { return kSmallU; }
uint32_t reprune_small_low_u() { return kSmallU2; }

namespace {
template <int E, int M, int LPR, int CPL>
cudaError_t launch_small_geom(const PruneArgs& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  const uint32_t blocks = std::min<uint32_t>((a.count + 3) / 4, 148u * 16u);
  if (a.small_u <= kSmallU2)
    reprune_small_kernel<E, M, LPR, CPL, kSmallU2><<<blocks, 128, 0, s>>>(a);
  else
    reprune_small_kernel<E, M, LPR, CPL, kSmallU><<<blocks, 128, 0, s>>>(a);
  return cudaGetLastError();
}
template <int E, int M>
cudaError_t launch_small_e(const PruneArgs& a, const Geometry& g, cudaStream_t s) {
  switch (g.lpr) {
    case 1: return launch_small_geom<E, M, 1, 1>(a, s);
    case 2: return launch_small_geom<E, M, 2, 1>(a, s);
    case 4: return launch_small_geom<E, M, 4, 1>(a, s);
    case 8: return launch_small_geom<E, M, 8, 1>(a, s);
    case 16: return launch_small_geom<E, M, 16, 1>(a, s);
    default:
      if (g.cpl == 1) return launch_small_geom<E, M, 32, 1>(a, s);
      if (g.cpl == 2) return launch_small_geom<E, M, 32, 2>(a, s);
      return launch_small_geom<E, M, 32, 4>(a, s);
  }
}
}  // namespace

cudaError_t launch_reprune_small(const PruneArgs& a, int elem, int metric, const Geometry& g, cudaStream_t s) {
  if (metric == kL2) return elem == kU8 ? launch_small_e<kU8, kL2>(a, g, s) : launch_small_e<kI8, kL2>(a, g, s);
  return elem == kU8 ? launch_small_e<kU8, kIP>(a, g, s) : launch_small_e<kI8, kIP>(a, g, s);
}

namespace {
template <int E, int M, int LPR, int CPL>
cudaError_t launch_nt(const PruneArgs& a, int threads, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  if (threads <= 32) {
    uint32_t Mcap = 32;
    while (Mcap < a.mcap && Mcap < (1u << 16)) Mcap <<= 1;
    const size_t smem = prune_smem_bytes(Mcap, a.R);
    auto k = prune_kernel<E, M, LPR, CPL, 32>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    k<<<a.count, 32, smem, s>>>(a, Mcap);
  } else {  // any length
    auto k = prune_chunked_kernel<E, M, LPR, CPL, 256>;
    const size_t cs = prune_chunked_smem(a.R);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(cs));
    if (e != cudaSuccess) return e;
    k<<<a.count, 256, cs, s>>>(a);
  }
  return cudaGetLastError();
}
template <int E, int M>
cudaError_t dispatch(const PruneArgs& a, const Geometry& g, int threads, cudaStream_t s) {
  switch (g.lpr) {
    case 1: return launch_nt<E, M, 1, 1>(a, threads, s);
    case 2: return launch_nt<E, M, 2, 1>(a, threads, s);
    case 4: return launch_nt<E, M, 4, 1>(a, threads, s);
    case 8: return launch_nt<E, M, 8, 1>(a, threads, s);
    case 16: return launch_nt<E, M, 16, 1>(a, threads, s);
    default:
      if (g.cpl == 1) return launch_nt<E, M, 32, 1>(a, threads, s);
      if (g.cpl == 2) return launch_nt<E, M, 32, 2>(a, threads, s);
      return launch_nt<E, M, 32, 4>(a, threads, s);
  }
}
}  // namespace

// One lane per list, rows streamed through a D-deep register ring: row i + D
// is loaded while candidate i is decided (selected or not), so the walk's bit
// tests do not wait on memory. W/4 16-byte loads per row; D * W registers of
// ring (64 at the depths used).
template <int W, int D>
__global__ void __launch_bounds__(128)
    prune_walk_ring_kernel(const PruneArgs a, const MmaLayout ly, const uint32_t* hand, uint32_t l0,
                           uint32_t lcount) {
  constexpr int Q = W / 4;  // uint4 per cull row
  const uint32_t rel = blockIdx.x * blockDim.x + threadIdx.x;
  if (rel >= lcount) return;
  const uint32_t li = l0 + rel;
  const uint32_t l = a.list_index ? a.list_index[li] : li;
  const uint32_t m = a.lengths[l];
  if (m < a.mmin || m > a.mcap) return;
  const uint32_t p = a.points[l];
  const uint32_t R = a.R;
  uint32_t* orow = a.out_rows ? a.out_rows + uint64_t(l) * R : a.out_adj + uint64_t(p - a.out_base) * R;
  const uint32_t* in = hand + size_t(rel) * ly.stride;
  const uint32_t m2 = in[0];
  const uint32_t* ids = in + 4;
  const uint32_t* zm = ids + ly.mc;
  const uint4* rows = reinterpret_cast<const uint4*>(zm + W);
  uint32_t cul[W];
#pragma unroll
  for (int w = 0; w < W; w++) cul[w] = 0u;
  uint4 ring[D][Q];
#pragma unroll
  for (int d = 0; d < D; d++)
#pragma unroll
    for (int q = 0; q < Q; q++)
      ring[d][q] = d < static_cast<int>(m2) ? __ldg(rows + size_t(d) * Q + q) : make_uint4(0u, 0u, 0u, 0u);
  uint32_t nsel = 0;
#pragma unroll
  for (int w = 0; w < W; w++) {
    if (32u * w >= m2 || nsel == R) break;
    const uint32_t zw = __ldg(zm + w);
    for (uint32_t g = 0; g < 32; g += D) {
      const uint32_t i0 = 32u * w + g;
      if (i0 >= m2 || nsel == R) break;
#pragma unroll
      for (int d = 0; d < D; d++) {
        const uint32_t i = i0 + d, b = g + d;
        uint4 cur[Q];
#pragma unroll
        for (int q = 0; q < Q; q++) {
          cur[q] = ring[d][q];
          ring[d][q] = i + D < m2 ? __ldg(rows + size_t(i + D) * Q + q) : make_uint4(0u, 0u, 0u, 0u);
        }
        if (i < m2 && nsel < R && !((cul[w] >> b) & 1u)) {  // prune.cpp:28-29
          orow[nsel] = __ldg(ids + i);
          nsel++;
          if (!((zw >> b) & 1u)) {  // prune.cpp:32: a zero-distance pick culls nothing
#pragma unroll
            for (int q = 0; q < Q; q++) {
              cul[4 * q + 0] |= cur[q].x;
              cul[4 * q + 1] |= cur[q].y;
              cul[4 * q + 2] |= cur[q].z;
              cul[4 * q + 3] |= cur[q].w;
            }
          }
        }
      }
    }
  }
  for (uint32_t i = nsel; i < R; i++) orow[i] = kNone;
  if (a.n_out) a.n_out[l] = nsel;
  if (a.spre && !a.out_rows) a.spre[p - a.out_base] = static_cast<uint8_t>(nsel < 255 ? nsel : 255);
}

template <int E, int M, int W>
cudaError_t launch_mma_w(const PruneArgs& a, const MmaLayout& ly, cudaStream_t s) {
  auto kp = a.rule == 0 ? prune_prep_kernel<E, M, W, 0> : prune_prep_kernel<E, M, W, 1>;
  cudaError_t e = cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ly.total));
  if (e != cudaSuccess) return e;
  // the hand-off region is reused chunk by chunk (~1 GiB)
  const uint64_t per = uint64_t(ly.stride) * 4;
  const uint32_t chunk = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(a.count, kHandoffMax / per)));
  uint32_t* hand = prune_handoff(a.hand, uint64_t(chunk) * per, s);
  if (!hand) return cudaErrorMemoryAllocation;
  const size_t walk_smem = size_t(kWalkWarps) * ly.mc * W * 4;
  if ((e = cudaFuncSetAttribute(prune_walk_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(walk_smem))) !=
      cudaSuccess)
    return e;
  // lane-per-list walks for the long insert-time lists (W >= 8: -8% prune
  // time at c1); the short re-prune lists stay on the warp walk with rows
  // staged in shared memory (the lane walk's dependent row loads made them
  // 6% slower). GANN_WALK_LANE=0/1 forces either.
  // walk: one lane per list through a register ring (measured at c1: -5% re-prune
  // time at W = 4, -8% insert prune time at W >= 8 against a warp per list);
  // GANN_WALK_RING=0 selects the warp walk
  const char* wr = std::getenv("GANN_WALK_RING");
  const bool ring = !(wr && *wr == '0');
  for (uint32_t l0 = 0; l0 < a.count; l0 += chunk) {
    const uint32_t n = std::min(chunk, a.count - l0);
    kp<<<n, PrepThreads<W>::value, ly.total, s>>>(a, ly, hand, l0, n);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (ring)
      prune_walk_ring_kernel<W, (W == 4 ? 16 : (W == 8 ? 8 : 4))><<<(n + 127) / 128, 128, 0, s>>>(a, ly, hand, l0, n);
    else
      prune_walk_kernel<W><<<(n + kWalkWarps - 1) / kWalkWarps, kWalkWarps * 32, walk_smem, s>>>(a, ly, hand, l0, n);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <int E, int M>
cudaError_t launch_mma(const PruneArgs& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  const MmaLayout ly = mma_layout(a.mcap, static_cast<uint32_t>(a.stride), a.R);
  if (ly.w == 4) return launch_mma_w<E, M, 4>(a, ly, s);
  if (ly.w == 8) return launch_mma_w<E, M, 8>(a, ly, s);
  return launch_mma_w<E, M, 16>(a, ly, s);
}

void prune_reserve(PruneHandoff* h, uint32_t lists, uint64_t stride, uint32_t R, cudaStream_t s) {
  // the largest hand-off a launch of `lists` lists (up to 512 candidates) asks for
  const uint64_t per = uint64_t(mma_layout(512, static_cast<uint32_t>(stride), R).stride) * 4;
  prune_handoff(h, std::min<uint64_t>(uint64_t(lists) * per, kHandoffMax / per * per), s);
}

namespace {
template <int E, int M, int LPR, int CPL>
void preload_prune_one() {
  touch_kernel(prune_kernel<E, M, LPR, CPL, 32>);
  if (E != kF32) {
    touch_kernel(reprune_small_kernel<E, M, LPR, CPL, kSmallU>);
    touch_kernel(reprune_small_kernel<E, M, LPR, CPL, kSmallU2>);
  }
  touch_kernel(prune_chunked_kernel<E, M, LPR, CPL, 256>);
  if (E != kF32) {
    touch_kernel(prune_prep_kernel<E, M, 4, 0>);
    touch_kernel(prune_prep_kernel<E, M, 4, 1>);
    touch_kernel(prune_prep_kernel<E, M, 8, 0>);
    touch_kernel(prune_prep_kernel<E, M, 8, 1>);
    touch_kernel(prune_prep_kernel<E, M, 16, 0>);
    touch_kernel(prune_prep_kernel<E, M, 16, 1>);
  }
}
template <int E, int M>
void preload_prune_geom(const Geometry& g) {
  switch (g.lpr) {
    case 1: return preload_prune_one<E, M, 1, 1>();
    case 2: return preload_prune_one<E, M, 2, 1>();
    case 4: return preload_prune_one<E, M, 4, 1>();
    case 8: return preload_prune_one<E, M, 8, 1>();
    case 16: return preload_prune_one<E, M, 16, 1>();
    default:
      if (g.cpl == 1) return preload_prune_one<E, M, 32, 1>();
      if (g.cpl == 2) return preload_prune_one<E, M, 32, 2>();
      return preload_prune_one<E, M, 32, 4>();
  }
}
}  // namespace

void preload_prune(int elem, int metric, const Geometry& g) {
  touch_kernel(bin_lists_kernel);
  touch_kernel(prune_walk_ring_kernel<4, 16>);
  touch_kernel(prune_walk_ring_kernel<8, 8>);
  touch_kernel(prune_walk_ring_kernel<16, 4>);
  if (metric == kL2) {
    if (elem == kU8) return preload_prune_geom<kU8, kL2>(g);
    if (elem == kI8) return preload_prune_geom<kI8, kL2>(g);
    return preload_prune_geom<kF32, kL2>(g);
  }
  if (elem == kU8) return preload_prune_geom<kU8, kIP>(g);
  if (elem == kI8) return preload_prune_geom<kI8, kIP>(g);
  return preload_prune_geom<kF32, kIP>(g);
}

bool prune_uses_mma(int elem, uint32_t mcap, uint64_t stride, uint32_t R) {
  if (elem == kF32 || mcap > 512 || mcap == 0) return false;
  return mma_layout(mcap, static_cast<uint32_t>(stride), R).total <= 200 * 1024;
}

cudaError_t launch_prune(const PruneArgs& a, int elem, int metric, const Geometry& g, int threads,
                         cudaStream_t s) {
  if (threads <= 32 && prune_uses_mma(elem, a.mcap, a.stride, a.R) && !std::getenv("GANN_NO_MMA")) {
    if (metric == kL2) return elem == kU8 ? launch_mma<kU8, kL2>(a, s) : launch_mma<kI8, kL2>(a, s);
    return elem == kU8 ? launch_mma<kU8, kIP>(a, s) : launch_mma<kI8, kIP>(a, s);
  }
  if (metric == kL2) {
    if (elem == kU8) return dispatch<kU8, kL2>(a, g, threads, s);
    if (elem == kI8) return dispatch<kI8, kL2>(a, g, threads, s);
    return dispatch<kF32, kL2>(a, g, threads, s);
  }
  if (elem == kU8) return dispatch<kU8, kIP>(a, g, threads, s);
  if (elem == kI8) return dispatch<kI8, kIP>(a, g, threads, s);
  return dispatch<kF32, kIP>(a, g, threads, s);
}

GANN_CHECK_READER(check_line_prune)

}  // namespace gann
