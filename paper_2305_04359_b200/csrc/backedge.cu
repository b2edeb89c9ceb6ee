// backedge.cu — phase 2 of a build batch: group the reverse pairs by target
// and merge them into the targets' out-lists (sm_100a).
//
// Behaviour contract: graphann::group_by_key (src/semisort.cpp:15-73) followed
// by graphann::apply_back_edges (src/builder_common.cpp:109-140), SURVEY.md
// §B.3 item 5: for each target t, with its new sources in pair order,
// M = N(t) ++ [sources not already in M]; |M| <= R -> N(t) = M, otherwise
// N(t) = alpha_prune(t, M with fresh d(t, .)).
//
// GPU semisort. A counting group-by instead of a comparison sort:
//   count    one atomicAdd per pair on a per-vertex counter (n words, kept
//            zero between batches); the first pair of a target claims a group
//            id (warp-aggregated);
//   offsets  each group bump-allocates its slot range (warp-aggregated atomics)
//            - group order is irrelevant, as in the reference's hash buckets;
//   scatter  one atomicAdd per pair on its group cursor writes the pair's
//            ordinal (its position in the pair stream) into the group range;
//   merge    one CTA per group sorts its ordinals in shared memory, which
//            restores the input order inside the group exactly (the
//            reference's per-bucket sort by (key, input index)), then merges,
//            dedupes and either writes the row or stages the list and its
//            distances for the prune kernel.
// Groups are size-binned: 32-thread CTAs for <= small_group_cap sources,
// 512-thread CTAs for hubs up to big_group_cap.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace gann {

namespace {

__device__ __forceinline__ uint32_t pair_target(const BackEdgeArgs& a, uint64_t e) {
  if (a.ptarget) return a.ptarget[e * a.pstride];
  const uint64_t b = e / a.R, i = e - b * a.R;
  return a.adj[uint64_t(a.bsrc[b] - a.base) * a.R + i];
}
__device__ __forceinline__ uint32_t pair_source(const BackEdgeArgs& a, uint64_t e) {
  if (a.psource) return a.psource[e];
  return a.bsrc[e / a.R];
}

// Warp-aggregated atomicAdd on a u64 counter: every active lane gets its own
// exclusive offset.
__device__ __forceinline__ unsigned long long warp_bump(unsigned long long* ctr, uint32_t v) {
  const uint32_t mask = __activemask();
  const int lane = threadIdx.x & 31;
  uint32_t incl = v;
  // inclusive scan over active lanes (inactive lanes contribute 0)
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(mask, incl, o);
    if (lane >= o && ((mask >> (lane - o)) & 1u)) incl += y;
  }
  const int leader = 31 - __clz(mask);
  unsigned long long base = 0;
  const uint32_t total = __shfl_sync(mask, incl, leader);
  if (lane == leader) base = atomicAdd(ctr, static_cast<unsigned long long>(total));
  base = __shfl_sync(mask, base, leader);
  return base + incl - v;
}

__global__ void be_count_kernel(const BackEdgeArgs a) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < a.npairs; e += stride) {
    const uint32_t t = pair_target(a, e);
    if (t == kNone) continue;
    const uint32_t old = atomicAdd(a.tcount + (t - a.base), 1u);
    if (old == 0) {
      const uint32_t g = static_cast<uint32_t>(atomicAdd(a.counters + kCntGroups, 1ull));
      a.tgroup[t - a.base] = g;
      a.gtarget[g] = t;
    }
  }
}

__global__ void be_offsets_kernel(const BackEdgeArgs a, const uint32_t ng) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  // whole warps stay converged for the aggregated bumps
  const bool valid = g < ng;
  const uint32_t c = valid ? a.tcount[a.gtarget[g] - a.base] : 0u;
  const unsigned long long o = warp_bump(a.counters + kCntPairsCursor, c);
  const unsigned long long p = warp_bump(a.counters + kCntPruneCursor, valid ? c + a.R : 0u);
  // one atomic per warp for the largest group (a per-thread atomicMax on one
  // address serialises ~n_groups operations in L2)
  const uint32_t wmax = __reduce_max_sync(0xFFFFFFFFu, c);
  if ((threadIdx.x & 31) == 0 && wmax) atomicMax(a.counters + kCntMaxGroup, static_cast<unsigned long long>(wmax));
  if (!valid) return;
  a.gcnt[g] = c;
  a.goff[g] = o;
  a.poff[g] = p;
  a.gcursor[g] = 0;
  if (c > a.small_group_cap) {
    const uint32_t i = static_cast<uint32_t>(atomicAdd(a.counters + kCntBig, 1ull));
    a.big_groups[i] = g;
  }
}

__global__ void be_scatter_kernel(const BackEdgeArgs a) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < a.npairs; e += stride) {
    const uint32_t t = pair_target(a, e);
    if (t == kNone) continue;
    const uint32_t g = a.tgroup[t - a.base];
    const uint32_t pos = atomicAdd(a.gcursor + g, 1u);
    GANN_CHECK(pos < a.gcnt[g] && a.goff[g] + pos < a.npairs);
    a.gsrc[a.goff[g] + pos] = a.pordinal ? a.pordinal[e * a.pstride] : static_cast<uint32_t>(e);
  }
}

template <int NT>
__device__ __forceinline__ void cta_sync() {
  if (NT == 32) __syncwarp(); else __syncthreads();
}

template <int NT>
__device__ void cta_sort_u32(uint32_t* v, uint32_t Mp) {
  for (uint32_t k = 2; k <= Mp; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < Mp; i += NT) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const uint32_t x = v[i], y = v[ixj];
          if ((x > y) == ((i & k) == 0)) {
            v[i] = y;
            v[ixj] = x;
          }
        }
      }
      cta_sync<NT>();
    }
  }
}

// Exclusive rank of flag among [0, n) for a CTA, chunked; calls f(i, rank) for set flags.
template <int NT, class F>
__device__ __forceinline__ uint32_t cta_stable_ranks(const uint8_t* flag, uint32_t n,
                                                     uint32_t* warp_tot, F&& f) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t total = 0;
  for (uint32_t b0 = 0; b0 < n; b0 += NT) {
    const uint32_t i = b0 + tid;
    const bool on = i < n && flag[i];
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, on);
    const uint32_t off = __popc(bal & ((1u << lane) - 1u));
    if (NT == 32) {
      if (on) f(i, total + off);
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
      if (on) f(i, total + before + off);
      total += all;
      __syncthreads();
    }
  }
  return total;
}

// MODE 0: merge into the graph (apply_back_edges). MODE 1: write the grouped
// pairs (group_by_key) to out_keys/out_vals at the group's slot range.
template <int E, int M, int LPR, int CPL, int NT, int MODE>
__global__ void __launch_bounds__(NT)
    be_merge_kernel(const BackEdgeArgs a, const uint32_t count, const uint32_t* glist,
                    const uint32_t cap, uint32_t* out_keys, uint32_t* out_vals) {
  using Op = DistOp<E, M>;
  constexpr int GROUPS = NT / LPR;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t warp_tot[NT / 32];
  __shared__ uint32_t sh_deg;
  uint32_t Cp = 32;
  while (Cp < cap) Cp <<= 1;
  uint32_t* ord = reinterpret_cast<uint32_t*>(smem);
  uint32_t* row = ord + Cp;
  uint8_t* kf = reinterpret_cast<uint8_t*>(row + a.R);
  const int tid = threadIdx.x;
  const uint32_t R = a.R;
  const uint32_t nch = static_cast<uint32_t>(a.stride >> 4);
  // re-prune list slots: one warp collects up to 32 group ids and claims
  // their slots with one atomic (a per-group atomic on one counter serialises
  // millions of operations per batch in L2)
  uint32_t pend = 0, npend = 0;
  auto flush_small = [&]() {
    unsigned long long base = 0;
    if (tid == 0) base = atomicAdd(a.counters + kCntPruneSmall, static_cast<unsigned long long>(npend));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (static_cast<uint32_t>(tid) < npend) a.plist_small[base + tid] = pend;
    npend = 0;
  };
  auto push_small = [&](uint32_t gg) {
    if (NT == 32) {
      if (static_cast<uint32_t>(tid) == npend) pend = gg;
      if (++npend == 32) flush_small();
    } else if (tid == 0) {
      const uint32_t i = static_cast<uint32_t>(atomicAdd(a.counters + kCntPruneSmall, 1ull));
      a.plist_small[i] = gg;
    }
  };

  for (uint32_t gi = blockIdx.x; gi < count; gi += gridDim.x) {
    const uint32_t g = glist ? glist[gi] : gi;
    const uint32_t c = a.gcnt[g];
    if (!glist && c > a.small_group_cap) continue;  // a hub: the big launch owns it
    if (c > cap) {
      if (tid == 0) atomicAdd(a.counters + kCntTooBig, 1ull);
      continue;
    }
    const uint32_t t = a.gtarget[g];
    const uint64_t go = a.goff[g];
    uint32_t* trow = a.adj + uint64_t(t - a.base) * R;
    uint32_t* pid = a.pid + a.poff[g];
    uint32_t nm;
    if (NT == 32 && c <= 32 && R <= 64) {
      // one warp, registers: rank-sort the ordinals (distinct), the row as two
      // ids per lane, each source tested against the row with one ballot
      const int lane = tid;
      const uint32_t FULL = 0xFFFFFFFFu;
      const uint32_t o = static_cast<uint32_t>(lane) < c ? a.gsrc[go + lane] : 0xFFFFFFFFu;
      uint32_t rk = 0;
      for (uint32_t j = 0; j < c; j++) rk += __shfl_sync(FULL, o, j) < o ? 1u : 0u;
      if (static_cast<uint32_t>(lane) < c) ord[rk] = o;  // input order inside the group (semisort.cpp:58-63)
      __syncwarp();
      if (MODE == 1) {
        const uint32_t key = a.key_of_target ? a.key_of_target[t] : t;
        if (static_cast<uint32_t>(lane) < c) {
          out_keys[go + lane] = key;
          out_vals[go + lane] = pair_source(a, ord[lane]);
        }
        __syncwarp();
        if (lane == 0) a.tcount[t - a.base] = 0;
        continue;
      }
      const uint32_t src = static_cast<uint32_t>(lane) < c ? pair_source(a, ord[lane]) : kNone;
      const uint32_t r0 = static_cast<uint32_t>(lane) < R ? trow[lane] : kNone;
      const uint32_t r1 = static_cast<uint32_t>(lane) + 32 < R ? trow[lane + 32] : kNone;
      const uint32_t deg = __popc(__ballot_sync(FULL, r0 != kNone)) + __popc(__ballot_sync(FULL, r1 != kNone));
      // first occurrence wins (builder_common.cpp:124-128)
      uint32_t keepmask = 0;
      for (uint32_t i = 0; i < c; i++) {
        const uint32_t si = __shfl_sync(FULL, src, i);
        bool dup = __ballot_sync(FULL, r0 == si || r1 == si) != 0;
        if (!a.sources_distinct) dup = dup || __ballot_sync(FULL, static_cast<uint32_t>(lane) < i && src == si) != 0;
        keepmask |= dup ? 0u : (1u << i);
      }
      if (static_cast<uint32_t>(lane) < deg) pid[lane] = r0;
      if (static_cast<uint32_t>(lane) + 32 < deg) pid[lane + 32] = r1;
      GANN_CHECK(!((keepmask >> lane) & 1u) || deg + __popc(keepmask & ((1u << lane) - 1u)) < a.R + c);
      if ((keepmask >> lane) & 1u) pid[deg + __popc(keepmask & ((1u << lane) - 1u))] = src;
      nm = deg + __popc(keepmask);
      __syncwarp();
    } else {
      uint32_t Mp = 32;
      while (Mp < c) Mp <<= 1;
      for (uint32_t i = tid; i < Mp; i += NT) ord[i] = i < c ? a.gsrc[go + i] : 0xFFFFFFFFu;
      cta_sync<NT>();
      cta_sort_u32<NT>(ord, Mp);  // input order inside the group (semisort.cpp:58-63)
      if (MODE == 1) {
        const uint32_t key = a.key_of_target ? a.key_of_target[t] : t;
        for (uint32_t i = tid; i < c; i += NT) {
          out_keys[go + i] = key;
          out_vals[go + i] = pair_source(a, ord[i]);
        }
        cta_sync<NT>();
        if (tid == 0) a.tcount[t - a.base] = 0;
        continue;
      }
      for (uint32_t i = tid; i < c; i += NT) ord[i] = pair_source(a, ord[i]);
      if (tid == 0) sh_deg = 0;
      cta_sync<NT>();
      for (uint32_t i = tid; i < R; i += NT) {
        const uint32_t v = trow[i];
        row[i] = v;
        if (v != kNone) atomicAdd(&sh_deg, 1u);
      }
      cta_sync<NT>();
      const uint32_t deg = sh_deg;
      // first occurrence wins (builder_common.cpp:124-128)
      for (uint32_t i = tid; i < c; i += NT) {
        const uint32_t s = ord[i];
        bool keep = true;
        for (uint32_t j = 0; j < deg && keep; j++) keep = row[j] != s;
        if (!a.sources_distinct)
          for (uint32_t j = 0; j < i && keep; j++) keep = ord[j] != s;
        kf[i] = keep ? 1 : 0;
      }
      cta_sync<NT>();
      for (uint32_t i = tid; i < deg; i += NT) pid[i] = row[i];
      const uint32_t kept = cta_stable_ranks<NT>(kf, c, warp_tot, [&](uint32_t i, uint32_t r) {
        pid[deg + r] = ord[i];
      });
      nm = deg + kept;
      cta_sync<NT>();
    }
    if (nm <= R) {  // builder_common.cpp:129-131
      for (uint32_t i = tid; i < R; i += NT) trow[i] = i < nm ? pid[i] : kNone;
    } else if (nm <= a.prune_small_cap && !a.small_dists) {
      // the tensor-core prune gathers these rows anyway and computes d(t, .) itself
      if (tid == 0) a.plen[g] = nm;
      push_small(g);
    } else {  // stage for alpha_prune with fresh distances (:133-138)
      const int sub = tid & (LPR - 1), grp = tid / LPR;
      uint4 tr[CPL];
      const uint8_t* tp = a.data + uint64_t(t) * a.stride;
#pragma unroll
      for (int cc = 0; cc < CPL; cc++) {
        const uint32_t ch = sub + cc * LPR;
        tr[cc] = ch < nch ? __ldg(reinterpret_cast<const uint4*>(tp) + ch) : make_uint4(0, 0, 0, 0);
      }
      float* pd = a.pdist + a.poff[g];
      constexpr int U = 4;
      for (uint32_t b0 = 0; b0 < nm; b0 += GROUPS * U) {
        uint4 x[U][CPL];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const uint32_t r = b0 + u * GROUPS + grp;
          const uint32_t id = r < nm ? pid[r] : 0u;
          const uint8_t* rp = a.data + uint64_t(id) * a.stride;
#pragma unroll
          for (int cc = 0; cc < CPL; cc++) {
            const uint32_t ch = sub + cc * LPR;
            x[u][cc] = (r < nm && ch < nch) ? __ldg(reinterpret_cast<const uint4*>(rp) + ch)
                                           : make_uint4(0, 0, 0, 0);
          }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
          typename Op::acc_t acc = Op::zero();
#pragma unroll
          for (int cc = 0; cc < CPL; cc++) acc = Op::chunk(tr[cc], x[u][cc], acc);
          acc = group_sum<LPR>(acc);
          const uint32_t r = b0 + u * GROUPS + grp;
          if (sub == 0 && r < nm) pd[r] = Op::finish(acc);
        }
      }
      if (tid == 0) a.plen[g] = nm;
      if (nm <= a.prune_small_cap) {
        push_small(g);
      } else if (tid == 0) {
        const uint32_t i = static_cast<uint32_t>(atomicAdd(a.counters + kCntPruneBig, 1ull));
        a.plist_big[i] = g;
      }
    }
    cta_sync<NT>();
    if (tid == 0) a.tcount[t - a.base] = 0;
  }
  if (NT == 32 && npend) flush_small();
}

// Hubs of the batch form (more sources than the small path handles, so the
// merged list certainly exceeds R): the list goes to alpha_prune, which sorts
// it by (dist, id), so pair order is irrelevant and no ordinal sort is needed.
// Sources are distinct per target in the batch form (each inserted point
// contributes at most one pair per target), so only the row check remains.
template <int E, int M, int LPR, int CPL, int NT>
__global__ void __launch_bounds__(NT)
    be_merge_hub_kernel(const BackEdgeArgs a, const uint32_t nbig) {
  using Op = DistOp<E, M>;
  constexpr int GROUPS = NT / LPR;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t sh_deg, sh_kept;
  uint32_t* row = reinterpret_cast<uint32_t*>(smem);
  const int tid = threadIdx.x;
  const uint32_t R = a.R;
  const uint32_t nch = static_cast<uint32_t>(a.stride >> 4);
  for (uint32_t gi = blockIdx.x; gi < nbig; gi += gridDim.x) {
    const uint32_t g = a.big_groups[gi];
    const uint32_t c = a.gcnt[g];
    const uint32_t t = a.gtarget[g];
    const uint64_t go = a.goff[g];
    uint32_t* trow = a.adj + uint64_t(t - a.base) * R;
    if (tid == 0) {
      sh_deg = 0;
      sh_kept = 0;
    }
    __syncthreads();
    for (uint32_t i = tid; i < R; i += NT) {
      const uint32_t v = trow[i];
      row[i] = v;
      if (v != kNone) atomicAdd(&sh_deg, 1u);
    }
    __syncthreads();
    const uint32_t deg = sh_deg;
    uint32_t* pid = a.pid + a.poff[g];
    for (uint32_t i = tid; i < deg; i += NT) pid[i] = row[i];
    for (uint32_t i = tid; i < c; i += NT) {
      const uint32_t s = pair_source(a, a.gsrc[go + i]);
      bool keep = true;
      for (uint32_t j = 0; j < deg && keep; j++) keep = row[j] != s;
      if (keep) pid[deg + atomicAdd(&sh_kept, 1u)] = s;
    }
    __syncthreads();
    const uint32_t nm = deg + sh_kept;
    const int sub = tid & (LPR - 1), grp = tid / LPR;
    uint4 tr[CPL];
    const uint8_t* tp = a.data + uint64_t(t) * a.stride;
#pragma unroll
    for (int cc = 0; cc < CPL; cc++) {
      const uint32_t ch = sub + cc * LPR;
      tr[cc] = ch < nch ? __ldg(reinterpret_cast<const uint4*>(tp) + ch) : make_uint4(0, 0, 0, 0);
    }
    float* pd = a.pdist + a.poff[g];
    constexpr int U = 4;
    for (uint32_t b0 = 0; b0 < nm; b0 += GROUPS * U) {
      uint4 x[U][CPL];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const uint32_t r = b0 + u * GROUPS + grp;
        const uint32_t id = r < nm ? pid[r] : 0u;
        const uint8_t* rp = a.data + uint64_t(id) * a.stride;
#pragma unroll
        for (int cc = 0; cc < CPL; cc++) {
          const uint32_t ch = sub + cc * LPR;
          x[u][cc] = (r < nm && ch < nch) ? __ldg(reinterpret_cast<const uint4*>(rp) + ch)
                                         : make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        typename Op::acc_t acc = Op::zero();
#pragma unroll
        for (int cc = 0; cc < CPL; cc++) acc = Op::chunk(tr[cc], x[u][cc], acc);
        acc = group_sum<LPR>(acc);
        const uint32_t r = b0 + u * GROUPS + grp;
        if (sub == 0 && r < nm) pd[r] = Op::finish(acc);
      }
    }
    if (tid == 0) {
      a.plen[g] = nm;
      atomicMax(a.counters + kCntMaxMerged, static_cast<unsigned long long>(nm));
      if (nm <= R) atomicAdd(a.counters + kCntTooBig, 1ull);  // cannot happen (c > R); flagged
      const uint32_t i = static_cast<uint32_t>(atomicAdd(a.counters + kCntPruneBig, 1ull));
      a.plist_big[i] = g;
      a.tcount[t - a.base] = 0;
    }
    __syncthreads();
  }
}

template <int E, int M, int LPR, int CPL, int MODE>
cudaError_t merge_launch(const BackEdgeArgs& a, uint32_t ng, uint32_t nbig, uint32_t* ok,
                         uint32_t* ov, cudaStream_t s) {
  if (ng > 0) {
    auto k = be_merge_kernel<E, M, LPR, CPL, 32, MODE>;
    const size_t smem = backedge_merge_smem(a.small_group_cap, a.R);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    // resident one-warp CTAs walking the groups (grid-stride) rather than one
    // CTA per group: millions of tiny CTAs per batch cost their launch, and a
    // warp with several groups claims re-prune slots 32 groups per atomic
    uint32_t grid = ng;
    const char* pg = std::getenv("GANN_MERGE_GRID");
    if (!(pg && *pg == '0')) {
      int dev = 0, sms = 0, per_sm = 0;
      if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
      if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
      if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32, smem)) != cudaSuccess) return e;
      grid = std::min<uint32_t>(ng, static_cast<uint32_t>(std::max(1, per_sm) * sms));
    }
    k<<<grid, 32, smem, s>>>(a, ng, nullptr, a.small_group_cap, ok, ov);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (nbig > 0 && MODE == 0 && a.sources_distinct) {
    auto k = be_merge_hub_kernel<E, M, LPR, CPL, 512>;
    const size_t smem = size_t(a.R) * 4;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    k<<<nbig, 512, smem, s>>>(a, nbig);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  } else if (nbig > 0) {
    auto k = be_merge_kernel<E, M, LPR, CPL, 512, MODE>;
    const size_t smem = backedge_merge_smem(a.big_group_cap, a.R);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    k<<<nbig, 512, smem, s>>>(a, nbig, a.big_groups, a.big_group_cap, ok, ov);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <int E, int M, int MODE>
cudaError_t merge_geom(const BackEdgeArgs& a, uint32_t ng, uint32_t nbig, const Geometry& g,
                       uint32_t* ok, uint32_t* ov, cudaStream_t s) {
  switch (g.lpr) {
    case 1: return merge_launch<E, M, 1, 1, MODE>(a, ng, nbig, ok, ov, s);
    case 2: return merge_launch<E, M, 2, 1, MODE>(a, ng, nbig, ok, ov, s);
    case 4: return merge_launch<E, M, 4, 1, MODE>(a, ng, nbig, ok, ov, s);
    case 8: return merge_launch<E, M, 8, 1, MODE>(a, ng, nbig, ok, ov, s);
    case 16: return merge_launch<E, M, 16, 1, MODE>(a, ng, nbig, ok, ov, s);
    default:
      if (g.cpl == 1) return merge_launch<E, M, 32, 1, MODE>(a, ng, nbig, ok, ov, s);
      if (g.cpl == 2) return merge_launch<E, M, 32, 2, MODE>(a, ng, nbig, ok, ov, s);
      return merge_launch<E, M, 32, 4, MODE>(a, ng, nbig, ok, ov, s);
  }
}

__global__ void hash_keys_kernel(const uint32_t* keys, uint64_t m, uint32_t* table, uint32_t tbits,
                                 uint32_t* slots) {
  const uint32_t mask = (1u << tbits) - 1u;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < m; e += stride) {
    const uint32_t k = keys[e];
    uint32_t s = static_cast<uint32_t>(mix64(k)) & mask;
    while (true) {
      const uint32_t old = atomicCAS(table + s, kNone, k);
      if (old == kNone || old == k) break;
      s = (s + 1) & mask;
    }
    slots[e] = s;
  }
}

__global__ void part_count_kernel(const uint32_t* adj, uint32_t base, uint32_t R, const uint32_t* ids,
                                  uint32_t K, uint32_t P, unsigned long long* counts) {
  const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= uint64_t(K) * R) return;
  const uint32_t k = static_cast<uint32_t>(e / R), i = static_cast<uint32_t>(e - uint64_t(k) * R);
  const uint32_t t = adj[uint64_t(ids[k] - base) * R + i];
  if (t != kNone) atomicAdd(counts + t / P, 1ull);
}

__global__ void part_scatter_kernel(const uint32_t* adj, uint32_t base, uint32_t R, const uint32_t* ids,
                                    const uint32_t* bo, uint32_t K, uint32_t P, unsigned long long* cursors,
                                    uint32_t* out) {
  const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= uint64_t(K) * R) return;
  const uint32_t k = static_cast<uint32_t>(e / R), i = static_cast<uint32_t>(e - uint64_t(k) * R);
  const uint32_t t = adj[uint64_t(ids[k] - base) * R + i];
  if (t == kNone) return;
  const unsigned long long pos = atomicAdd(cursors + t / P, 1ull);
  out[2 * pos] = t;
  out[2 * pos + 1] = bo[k] * R + i;  // the pair's position in the batch's concatenation order
}

}  // namespace

cudaError_t part_pairs_count(const uint32_t* adj_local, uint32_t base, uint32_t R, const uint32_t* ids,
                             uint32_t K, uint32_t P, unsigned long long* counts, cudaStream_t s) {
  const uint64_t n = uint64_t(K) * R;
  if (n == 0) return cudaSuccess;
  part_count_kernel<<<static_cast<uint32_t>((n + 255) / 256), 256, 0, s>>>(adj_local, base, R, ids, K, P, counts);
  return cudaGetLastError();
}

cudaError_t part_pairs_scatter(const uint32_t* adj_local, uint32_t base, uint32_t R, const uint32_t* ids,
                               const uint32_t* bo, uint32_t K, uint32_t P, unsigned long long* cursors,
                               uint32_t* out_pairs, cudaStream_t s) {
  const uint64_t n = uint64_t(K) * R;
  if (n == 0) return cudaSuccess;
  part_scatter_kernel<<<static_cast<uint32_t>((n + 255) / 256), 256, 0, s>>>(adj_local, base, R, ids, bo, K, P,
                                                                             cursors, out_pairs);
  return cudaGetLastError();
}

cudaError_t launch_hash_keys(const uint32_t* keys, uint64_t m, uint32_t* table, uint32_t tbits,
                             uint32_t* slots, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(table, 0xFF, (size_t(1) << tbits) * 4, s);
  if (e != cudaSuccess || m == 0) return e;
  hash_keys_kernel<<<static_cast<uint32_t>(std::min<uint64_t>((m + 255) / 256, 148 * 32)), 256, 0, s>>>(
      keys, m, table, tbits, slots);
  return cudaGetLastError();
}

size_t backedge_merge_smem(uint32_t cap, uint32_t R) {
  uint32_t Cp = 32;
  while (Cp < cap) Cp <<= 1;
  size_t b = size_t(Cp) * 4 + size_t(R) * 4 + size_t(Cp);
  return (b + 15) & ~size_t(15);
}

cudaError_t backedge_count(const BackEdgeArgs& a, cudaStream_t s) {
  if (a.npairs == 0) return cudaSuccess;
  const uint64_t blocks = (a.npairs + 255) / 256;
  be_count_kernel<<<static_cast<uint32_t>(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t backedge_offsets(const BackEdgeArgs& a, uint32_t ng, cudaStream_t s) {
  if (ng == 0) return cudaSuccess;
  be_offsets_kernel<<<(ng + 255) / 256, 256, 0, s>>>(a, ng);
  return cudaGetLastError();
}

cudaError_t backedge_scatter(const BackEdgeArgs& a, cudaStream_t s) {
  if (a.npairs == 0) return cudaSuccess;
  const uint64_t blocks = (a.npairs + 255) / 256;
  be_scatter_kernel<<<static_cast<uint32_t>(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t backedge_merge(const BackEdgeArgs& a, uint32_t ng, uint32_t nbig, int elem, int metric,
                           const Geometry& g, cudaStream_t s) {
  if (metric == kL2) {
    if (elem == kU8) return merge_geom<kU8, kL2, 0>(a, ng, nbig, g, nullptr, nullptr, s);
    if (elem == kI8) return merge_geom<kI8, kL2, 0>(a, ng, nbig, g, nullptr, nullptr, s);
    return merge_geom<kF32, kL2, 0>(a, ng, nbig, g, nullptr, nullptr, s);
  }
  if (elem == kU8) return merge_geom<kU8, kIP, 0>(a, ng, nbig, g, nullptr, nullptr, s);
  if (elem == kI8) return merge_geom<kI8, kIP, 0>(a, ng, nbig, g, nullptr, nullptr, s);
  return merge_geom<kF32, kIP, 0>(a, ng, nbig, g, nullptr, nullptr, s);
}

namespace {
template <int E, int M, int LPR, int CPL>
void preload_be_one() {
  touch_kernel(be_merge_kernel<E, M, LPR, CPL, 32, 0>);
  touch_kernel(be_merge_kernel<E, M, LPR, CPL, 512, 0>);
  touch_kernel(be_merge_hub_kernel<E, M, LPR, CPL, 512>);
}
template <int E, int M>
void preload_be_geom(const Geometry& g) {
  switch (g.lpr) {
    case 1: return preload_be_one<E, M, 1, 1>();
    case 2: return preload_be_one<E, M, 2, 1>();
    case 4: return preload_be_one<E, M, 4, 1>();
    case 8: return preload_be_one<E, M, 8, 1>();
    case 16: return preload_be_one<E, M, 16, 1>();
    default:
      if (g.cpl == 1) return preload_be_one<E, M, 32, 1>();
      if (g.cpl == 2) return preload_be_one<E, M, 32, 2>();
      return preload_be_one<E, M, 32, 4>();
  }
}
}  // namespace

void preload_backedge(int elem, int metric, const Geometry& g) {
  touch_kernel(be_count_kernel);
  touch_kernel(be_offsets_kernel);
  touch_kernel(be_scatter_kernel);
  if (metric == kL2) {
    if (elem == kU8) return preload_be_geom<kU8, kL2>(g);
    if (elem == kI8) return preload_be_geom<kI8, kL2>(g);
    return preload_be_geom<kF32, kL2>(g);
  }
  if (elem == kU8) return preload_be_geom<kU8, kIP>(g);
  if (elem == kI8) return preload_be_geom<kI8, kIP>(g);
  return preload_be_geom<kF32, kIP>(g);
}

cudaError_t backedge_write_groups(const BackEdgeArgs& a, uint32_t ng, uint32_t nbig,
                                  uint32_t* out_keys, uint32_t* out_vals, cudaStream_t s) {
  Geometry g{1, 1, 1};
  return merge_geom<kU8, kL2, 1>(a, ng, nbig, g, out_keys, out_vals, s);
}

GANN_CHECK_READER(check_line_backedge)

}  // namespace gann
