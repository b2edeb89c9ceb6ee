// search_batch.cuh — beam search with several expansions per step (sm_100a).
//
// Same contract as search_kernel (graphann::beam_search, src/search.cpp:62-131:
// identical ids, distances, |V| and visit order), for the Alg. 1 form
// {L, k = L, eps} in the fast visited mode with R <= 64. One warp per query.
//
// The reference expands one vertex per step: the first unexpanded beam key
// (src/search.cpp:96-103). Each such step is a chain of dependent memory round
// trips (adjacency row -> visited probes -> vector rows -> merge), and at large
// beams that chain, not bandwidth, set the old kernel's time (c1, L = 832: 0.14
// of the HBM peak at 20 resident warps per SM). Here a step takes the first
// EB unexpanded keys x_0 < x_1 < ... at once:
//   * their adjacency rows are loaded together, all neighbours are probed in
//     the visited table together (read only), and the fresh ones' rows are
//     gathered in one stream of passes;
//   * expansion f is what the reference would do next exactly when no new key
//     from expansions 0..f-1 lies below x_f (then x_f is still the first
//     unexpanded key). A surviving new key k from expansion e first breaks
//     expansion max(e + 1, #{f : x_f < k}); the smallest such index over all
//     survivors is P, and expansions 0..P-1 are committed: marked expanded,
//     appended to the visit list in order, their fresh ids entered into the
//     visited table, their survivors merged — in ONE merge, equal to the P
//     sequential merges because the beam is the top-L of everything pushed and
//     the L-th key only ever decreases. Expansions P.. are dropped unseen
//     (their ids were never entered into the table) and come up again;
//   * on c1 (10M x 128 u8, R = 64) ~88% of next-expansion guesses hold at L =
//     832 and a step of up to 8 commits ~5.5 expansions (CPU simulation on the
//     same generator: tools/sim_spec.py), so the chain and the merge's fixed
//     cost are paid once per ~5 expansions.
// The visited table is the per-warp region in global memory (L2-resident) of
// search_kernel's second level; exact-positive (u16 remainders of a bijective
// hash), so results never depend on it. Two rows of one step may both list a
// fresh id: both are gathered, and the merge drops the second of two equal
// survivor keys (measured: ~1% of candidates).
#pragma once

namespace gann {
namespace {

#ifndef GANN_BATCH_EB
#define GANN_BATCH_EB 4  // expansions per step (compile-time bound, <= 8)
#endif
#ifndef GANN_BATCH_MINB
#define GANN_BATCH_MINB 6  // resident 4-warp CTAs per SM the register budget targets
#endif

// The gather's 16-byte load (GANN_GATHER_LD: 0 ld.global.nc, 1 ld.global.cg, 2 nc + L1::no_allocate)
#ifndef GANN_GATHER_LD
#define GANN_GATHER_LD 0
#endif
__device__ __forceinline__ uint4 gather_ld(const uint4* p) {
#if GANN_GATHER_LD == 1
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
#elif GANN_GATHER_LD == 2
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
#else
  return __ldg(p);
#endif
}

// A visited-table bucket read (GANN_PROBE_LD: 0 ld.global.cg with the L2 policy, 1 atom.or 0 at L2,
// 2 ld.relaxed.gpu, 3 ld.volatile)
#ifndef GANN_PROBE_LD
#define GANN_PROBE_LD 0
#endif
__device__ __forceinline__ uint64_t probe_ld(const uint64_t* p, uint64_t pol) {
  uint64_t v;
#if GANN_PROBE_LD == 1
  asm volatile("atom.global.or.b64 %0, [%1], 0;" : "=l"(v) : "l"(p) : "memory");
#elif GANN_PROBE_LD == 2
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
#elif GANN_PROBE_LD == 3
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
#else
  asm volatile("ld.global.cg.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol) : "memory");
#endif
  return v;
}

// The visited table's buckets. Narrow (n <= 2^(log2 + 15)): four u16 slots per
// u64 bucket holding the 15-bit remainders of a bijective hash of the id, so a
// match is the same id (0xFFFF: empty); the bucket is the hash's upper bits.
// Wide (larger n, up to 2^32 - 2): two u32 slots holding whole ids (0xFFFFFFFF:
// empty). An insert shifts the bucket and drops its oldest slot.
__device__ __forceinline__ uint32_t tab_bucket(uint32_t id, bool wide, uint32_t mask, uint32_t log2) {
  const uint32_t h = id * 0x85EBCA6Bu;
  return wide ? h >> (32u - log2) : (h & mask) >> 15;
}
__device__ __forceinline__ bool tab_hit(uint64_t w, uint32_t id, bool wide) {
  if (wide) return static_cast<uint32_t>(w) == id || static_cast<uint32_t>(w >> 32) == id;
  const uint32_t rem = (id * 0x85EBCA6Bu) & 0x7FFFu;
  const uint32_t rr = rem | (rem << 16);
  // a u16 slot equal to rem <=> a zero half word in w ^ rr (exact as a yes/no:
  // a borrow only ever follows a true zero)
  const uint32_t y0 = static_cast<uint32_t>(w) ^ rr, y1 = static_cast<uint32_t>(w >> 32) ^ rr;
  return ((((y0 - 0x00010001u) & ~y0) | ((y1 - 0x00010001u) & ~y1)) & 0x80008000u) != 0u;
}
__device__ __forceinline__ uint64_t tab_insert(uint64_t w, uint32_t id, bool wide) {
  if (wide) return (w << 32) | id;
  return (w << 16) | ((id * 0x85EBCA6Bu) & 0x7FFFu);
}

// One gather pass (eval_pass) that also carries each row's expansion index
// next to its key.
template <class Op, int LPR, int CPL, int UU, bool FIT>
__device__ __forceinline__ void beval_pass(uint32_t b0, const uint32_t* ids, const uint8_t* ex, uint32_t m,
                                           uint32_t stride, const uint8_t* const (&cb)[CPL], const bool (&chv)[CPL],
                                           uint64_t* out, uint8_t* oute, const uint4 (&qr)[CPL], int sub, int grp,
                                           uint64_t worst, uint32_t& n_out, int lane) {
  const uint32_t rb = b0 + grp * UU;
  uint32_t id[UU];
  if (UU % 4 == 0) {
#pragma unroll
    for (int u = 0; u < UU; u += 4) {
      const uint4 v = *reinterpret_cast<const uint4*>(ids + rb + u);
      id[u] = v.x;
      if (u + 1 < UU) id[u + 1] = v.y;
      if (u + 2 < UU) id[u + 2] = v.z;
      if (u + 3 < UU) id[u + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int u = 0; u < UU; u++) id[u] = ids[rb + u];
  }
  uint4 x[UU][CPL];
#pragma unroll
  for (int u = 0; u < UU; u++) {
#pragma unroll
    for (int c = 0; c < CPL; c++) x[u][c] = gather_ld(row_chunk(cb[c], id[u], stride));
  }
  typename Op::acc_t acc[UU];
#pragma unroll
  for (int u = 0; u < UU; u++) {
    acc[u] = Op::zero();
#pragma unroll
    for (int c = 0; c < CPL; c++)
      if (FIT || chv[c]) acc[u] = Op::chunk(qr[c], x[u][c], acc[u]);
  }
  const typename Op::acc_t tot = transpose_reduce<LPR, UU>(acc, sub);
  const uint32_t r = rb + (sub & (UU - 1));
  uint64_t key = kMaxKey;
  if (sub < UU && r < m) key = make_bkey(Op::finish(tot), ids[r]);
  const bool keep = key < worst;
  const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
  if (keep) {
    const uint32_t o = n_out + __popc(bal & ((1u << lane) - 1u));
    GANN_CHECK(o < m);
    out[o] = key;
    oute[o] = ex[r];
  }
  n_out += __popc(bal);
}

template <class Op, int LPR, int CPL, bool FIT>
__device__ __forceinline__ uint32_t beval_rows(const uint8_t* __restrict__ data, uint32_t stride, uint32_t nch,
                                               const uint32_t* ids, const uint8_t* ex, uint32_t m, uint64_t* out,
                                               uint8_t* oute, const uint4 (&qr)[CPL], int lane, uint64_t worst) {
  constexpr int RPP = 32 / LPR;
  constexpr int U = Unroll<LPR, CPL>::U;
  const int sub = lane & (LPR - 1);
  const int grp = lane / LPR;
  bool chv[CPL];
  const uint8_t* cb[CPL];
#pragma unroll
  for (int c = 0; c < CPL; c++) {
    const uint32_t ch = static_cast<uint32_t>(sub + c * LPR);
    chv[c] = FIT || ch < nch;
    cb[c] = data + static_cast<size_t>(chv[c] ? ch : nch - 1) * 16;
  }
  uint32_t b0 = 0, n_out = 0;
  for (; b0 + RPP * U <= m; b0 += RPP * U)
    beval_pass<Op, LPR, CPL, U, FIT>(b0, ids, ex, m, stride, cb, chv, out, oute, qr, sub, grp, worst, n_out, lane);
  const uint32_t rem = m - b0;
  if (rem == 0) return n_out;
  if (U >= 8 && rem <= RPP * (U / 4))
    beval_pass<Op, LPR, CPL, (U >= 8 ? U / 4 : 1), FIT>(b0, ids, ex, m, stride, cb, chv, out, oute, qr, sub, grp, worst, n_out, lane);
  else if (U >= 4 && rem <= RPP * (U / 2))
    beval_pass<Op, LPR, CPL, (U >= 4 ? U / 2 : 1), FIT>(b0, ids, ex, m, stride, cb, chv, out, oute, qr, sub, grp, worst, n_out, lane);
  else
    beval_pass<Op, LPR, CPL, U, FIT>(b0, ids, ex, m, stride, cb, chv, out, oute, qr, sub, grp, worst, n_out, lane);
  return n_out;
}

}  // namespace

template <int E, int M, int LPR, int CPL, bool FIT>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, GANN_BATCH_MINB)
    search_batch_kernel(const SearchArgs a, const uint32_t per_warp, const uint32_t cm) {
  using Op = DistOp<E, M>;
  constexpr int EB = GANN_BATCH_EB;
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint32_t L = a.L, R = a.R;  // R <= 64 (host)
  const uint32_t Lp = (L + 31) & ~31u;
  const uint32_t nch = static_cast<uint32_t>(a.stride >> 4);
  const uint32_t stride32 = static_cast<uint32_t>(a.stride);
  uint8_t* base = smem + wib * per_warp;
  uint64_t* beam = reinterpret_cast<uint64_t*>(base);
  uint64_t* ck = beam + Lp;                                  // keys below the L-th, then the survivors
  uint32_t* cid = reinterpret_cast<uint32_t*>(ck + cm);      // fresh ids of the step
  uint32_t* epos = cid + cm;                                 // beam positions of the step's expansions (8 words, 16-byte aligned)
  uint32_t* bm = epos + 8;                                   // Lp bits: final positions of the survivors
  uint16_t* posb = reinterpret_cast<uint16_t*>(bm + Lp / 32);  // insertion points (L < 65536)
  uint8_t* cex = reinterpret_cast<uint8_t*>(posb + cm);      // expansion of a candidate; later rank -> survivor
  uint8_t* cke = cex + cm;                                   // expansion of a key; later the survivor's rank
  uint8_t* inv = cex;
  const uint32_t FULL = 0xFFFFFFFFu;

  // this warp's visited-table region (as search_kernel's second level)
  uint64_t* g2 = nullptr;
  uint32_t g2_region = kNone;
  uint64_t g2pol = 0;
  if (a.gtab_keep)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(g2pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(g2pol));
  // (a region per resident warp of two launches exists, so a free one is
  // found at once; the retries only cover a warp that has not released yet)
  for (uint32_t attempt = 0; lane == 0 && g2_region == kNone && attempt < (1u << 16); attempt++) {
    const uint32_t words = (a.gtab_regions + 31) / 32;
    const uint32_t w0 = (blockIdx.x * 32 + (threadIdx.x >> 5) + attempt) % words;
    for (uint32_t t = 0; t < words && g2_region == kNone; t++) {
      const uint32_t w = (w0 + t) % words;
      uint32_t cur = a.gtab_busy[w];
      while (cur != 0xFFFFFFFFu) {
        const int b = __ffs(~cur) - 1;
        if (w * 32 + b >= a.gtab_regions) break;
        const uint32_t old = atomicOr(a.gtab_busy + w, 1u << b);
        if (!(old & (1u << b))) {
          g2_region = w * 32 + b;
          break;
        }
        cur = old | (1u << b);
      }
    }
  }
  g2_region = __shfl_sync(FULL, g2_region, 0);
  if (g2_region == kNone) {  // cannot happen with the host's region count; loud if it does
    if (lane == 0) atomicAdd(a.overflow + 2, 1u);
    return;
  }
  g2 = a.gtab + (static_cast<uint64_t>(g2_region) << a.gtab_log2);
  const uint32_t g2mask = (1u << (a.gtab_log2 + 15)) - 1u;
  const bool wide = a.gtab_wide != 0;

  uint32_t q = 0;
  if (lane == 0) q = atomicAdd(a.next_query, 1u);
  q = __shfl_sync(FULL, q, 0);
  for (; q < a.nq;) {
#pragma unroll 1
    for (uint32_t i = lane; i < (1u << a.gtab_log2) / 2; i += 32)  // empty table: 0xFFFF is no remainder
      asm volatile("st.global.cg.L2::cache_hint.v4.u32 [%0], {%1, %1, %1, %1}, %2;"
                   :: "l"(reinterpret_cast<uint4*>(g2) + i), "r"(kNone), "l"(g2pol) : "memory");
    const uint8_t* qp = a.query_rows ? a.data + static_cast<uint64_t>(a.query_rows[q]) * a.stride
                                     : a.queries + static_cast<uint64_t>(q) * a.stride;
    const int sub = lane & (LPR - 1);
    uint4 qr[CPL];
#pragma unroll
    for (int c = 0; c < CPL; c++) {
      const uint32_t ch = sub + c * LPR;
      qr[c] = ch < nch ? __ldg(reinterpret_cast<const uint4*>(qp) + ch) : make_uint4(0, 0, 0, 0);
    }
    const uint32_t start = a.start_override ? a.start_override[q] : a.start;
#pragma unroll 1
    for (uint32_t i = lane; i < Lp / 32; i += 32) bm[i] = 0;
    cid[lane] = start;  // padded: whole passes
    cex[lane] = 0;
    __syncwarp();
    beval_rows<Op, LPR, CPL, FIT>(a.data, stride32, nch, cid, cex, 1, ck, cke, qr, lane, kMaxKey);
    __syncwarp();
    if (lane == 0) beam[0] = ck[0];
    uint32_t size = 1, nvis = 0, hint = 0;
    uint32_t eb = 1;  // expansions to try in the next step
    uint64_t evals = 1;
    uint32_t steps = 0, dropped = 0, nsurv = 0;
    __syncwarp();

    while (true) {
      // ---- the first eb unexpanded keys at or after hint ----
      uint32_t nsel = 0;
#pragma unroll 1
      for (uint32_t b0 = hint & ~31u; b0 < size && nsel < eb; b0 += 32) {
        const uint32_t i = b0 + lane;
        const bool un = i >= hint && i < size && (beam[i] & 1ull) == 0;
        const uint32_t bal = __ballot_sync(FULL, un);
        const uint32_t slot = nsel + __popc(bal & lanemask_lt(lane));
        if (un && slot < eb) epos[slot] = i;
        nsel += __popc(bal);
      }
      if (nsel == 0) break;
      nsel = min(nsel, eb);
      if (lane >= nsel && lane < 8) epos[lane] = kNone;  // no position: never below an insertion point
      __syncwarp();
      // lane f holds expansion f
      const uint32_t xpos = lane < nsel ? epos[lane] : kNone;
      const uint64_t xkey = lane < nsel ? beam[xpos] : kMaxKey;
      const uint32_t xid = bkey_id(xkey);
      const uint32_t x0 = __shfl_sync(FULL, xid, 0);

      // ---- their adjacency rows, then every neighbour's table bucket (read only) ----
      uint32_t nb[EB][2];
#pragma unroll
      for (int e = 0; e < EB; e++) {
        const uint32_t v = __shfl_sync(FULL, xid, e);
        nb[e][0] = kNone;
        nb[e][1] = kNone;
        if (e < nsel) {
          const uint32_t* row = graph_row(a.graph, v, R);
          if (lane < R) nb[e][0] = __ldg(row + lane);
          if (lane + 32 < R) nb[e][1] = __ldg(row + 32 + lane);
        }
      }
      uint64_t w[EB][2];
#pragma unroll
      for (int e = 0; e < EB; e++) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
          w[e][h] = 0ull;
          if (nb[e][h] != kNone) {
            const uint32_t bucket = tab_bucket(nb[e][h], wide, g2mask, a.gtab_log2);
            w[e][h] = probe_ld(g2 + bucket, g2pol);
          }
        }
      }
      // fresh ids, in expansion order then adjacency order; a step holds at
      // most cm of them (later expansions wait for the next step)
      uint32_t m = 0, nlive = nsel;
#pragma unroll
      for (int e = 0; e < EB; e++) {
        if (e < nlive) {
          bool fr[2];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            fr[h] = nb[e][h] != kNone && !tab_hit(w[e][h], nb[e][h], wide);
          }
          const uint32_t b0 = __ballot_sync(FULL, fr[0]), b1 = __ballot_sync(FULL, fr[1]);
          const uint32_t c = __popc(b0) + __popc(b1);
          if (e > 0 && m + c > cm) {
            nlive = e;
          } else {
            if (fr[0]) {
              const uint32_t o = m + __popc(b0 & lanemask_lt(lane));
              GANN_CHECK(o < cm);
              cid[o] = nb[e][0];
              cex[o] = static_cast<uint8_t>(e);
            }
            if (fr[1]) {
              const uint32_t o = m + __popc(b0) + __popc(b1 & lanemask_lt(lane));
              GANN_CHECK(o < cm);
              cid[o] = nb[e][1];
              cex[o] = static_cast<uint8_t>(e);
            }
            m += c;
          }
        }
      }
      nsel = nlive;

      // ---- distances; keys below the L-th beam key go to ck (c1 of them) ----
      uint32_t c1 = 0;
      if (m) {
        if (m + lane < ((m + 31) & ~31u)) cid[m + lane] = x0;  // pad to a whole pass
        __syncwarp();
        evals += m;
        const uint64_t worst = size == L ? beam[L - 1] : kMaxKey;
        c1 = beval_rows<Op, LPR, CPL, FIT>(a.data, stride32, nch, cid, cex, m, ck, cke, qr, lane, worst);
        __syncwarp();
      }

      // ---- insertion points; beam duplicates drop; the first expansion a survivor breaks ----
      uint32_t s = 0, pmin = nsel;
#pragma unroll 1
      for (uint32_t j0 = 0; j0 < c1; j0 += 32) {
        const uint32_t j = j0 + lane;
        bool keep = j < c1;
        const uint64_t k = keep ? ck[j] : kMaxKey;
        const uint32_t e = keep ? cke[j] : 0u;
        uint32_t pb = 0;
        if (keep) {
          pb = lower_bound_steps_u64(beam, size, k);
          if (pb < size && (beam[pb] | 1ull) == (k | 1ull)) keep = false;  // a re-evaluated beam key
        }
        if (keep) {
          // x_f < k  <=>  x_f's position is below k's insertion point
          const uint4 p0 = *reinterpret_cast<const uint4*>(epos), p1 = *reinterpret_cast<const uint4*>(epos + 4);
          const uint32_t g = (p0.x < pb) + (p0.y < pb) + (p0.z < pb) + (p0.w < pb) + (p1.x < pb) + (p1.y < pb) +
                             (p1.z < pb) + (p1.w < pb);
          pmin = min(pmin, max(e + 1u, g));
        }
        __syncwarp();  // this chunk's keys are read before the compaction overwrites them
        const uint32_t bal = __ballot_sync(FULL, keep);
        if (keep) {
          const uint32_t o = s + __popc(bal & lanemask_lt(lane));
          ck[o] = k;
          cke[o] = static_cast<uint8_t>(e);
          posb[o] = static_cast<uint16_t>(pb);
        }
        s += __popc(bal);
      }
      const uint32_t P = min(nsel, __reduce_min_sync(FULL, pmin));  // >= 1

      // ---- commit expansions 0..P-1 ----
      if (lane < P) {
        beam[xpos] = xkey | 1ull;
        if (a.vis_ids && nvis + lane < a.vcap) {
          a.vis_ids[static_cast<uint64_t>(q) * a.vcap + nvis + lane] = xid;
          a.vis_dists[static_cast<uint64_t>(q) * a.vcap + nvis + lane] = key_dist(xkey);
        }
      }
      nvis += P;
      steps++;
      dropped += nsel - P;
      const uint32_t xlast = __shfl_sync(FULL, xpos, P - 1);
      eb = a.batch_policy == 0 ? static_cast<uint32_t>(EB)
                               : (a.batch_policy == 2 && P == nsel ? static_cast<uint32_t>(EB) : min(static_cast<uint32_t>(EB), P + 1u));
      eb = min(eb, a.batch_eb);
      // their fresh ids enter the visited table (newest remainder in the low
      // half word). Up to 64 of them (the default step): the buckets are read
      // here and written at the end of the step, behind the merge, so the L2
      // round trip is not waited for (the next step's probes come after it)
      uint64_t tw[2] = {0ull, 0ull};
      uint32_t tb[2] = {kNone, kNone}, tr[2] = {0u, 0u};  // bucket, id
      if (m <= 64) {
#pragma unroll
        for (int t = 0; t < 2; t++) {
          const uint32_t j = static_cast<uint32_t>(t) * 32 + lane;
          if (j < m && cex[j] < P) {
            tr[t] = cid[j];
            tb[t] = tab_bucket(tr[t], wide, g2mask, a.gtab_log2);
            tw[t] = probe_ld(g2 + tb[t], g2pol);
          }
        }
      } else {
#pragma unroll 1
        for (uint32_t j0 = 0; j0 < m; j0 += 32) {
          const uint32_t j = j0 + lane;
          if (j < m && cex[j] < P) {
            const uint32_t bucket = tab_bucket(cid[j], wide, g2mask, a.gtab_log2);
            const uint64_t wv = probe_ld(g2 + bucket, g2pol);
            asm volatile("st.global.cg.L2::cache_hint.u64 [%0], %1, %2;" :: "l"(g2 + bucket), "l"(tab_insert(wv, cid[j], wide)), "l"(g2pol) : "memory");
          }
        }
      }
      auto table_commit = [&]() {
#pragma unroll
        for (int t = 0; t < 2; t++)
          if (tb[t] != kNone)
            asm volatile("st.global.cg.L2::cache_hint.u64 [%0], %1, %2;" :: "l"(g2 + tb[t]), "l"(tab_insert(tw[t], tr[t], wide)), "l"(g2pol) : "memory");
      };
      hint = xlast + 1;
      __syncwarp();
      // survivors of dropped expansions leave (kMaxKey sorts behind every key)
      uint32_t sreal = s;
      if (P < nsel) {
#pragma unroll 1
        for (uint32_t j0 = 0; j0 < s; j0 += 32) {
          const uint32_t j = j0 + lane;
          const bool drop = j < s && cke[j] >= P;
          if (drop) ck[j] = kMaxKey;
          sreal -= __popc(__ballot_sync(FULL, drop));
        }
        __syncwarp();
      }
      if (sreal == 0) {
        table_commit();
        continue;
      }

      // ---- survivors ranked ----
      // Fast path: ranks by a 32-bit window of the keys (cd, 4 per shared
      // load): the bits of key - (smallest distance word << 32) from the highest
      // differing distance bit down, i.e. the distance differences and as many
      // id bits as still fit. Survivors lie in a narrow distance band, so two
      // of them rarely share a window; when two collide on a rank slot the
      // exact pass below ranks by whole keys, where a collision is the second
      // of two equal keys (one id fresh in two rows of the step), which leaves.
      uint32_t* cd = cid;  // the fresh ids are dead: the survivors' windows
      {
        uint32_t dmin = 0xFFFFFFFFu, dmax = 0u;
#pragma unroll 1
        for (uint32_t j0 = 0; j0 < s; j0 += 32) {
          const uint32_t j = j0 + lane;
          const uint64_t k = j < s ? ck[j] : kMaxKey;
          if (k != kMaxKey) {
            dmin = min(dmin, static_cast<uint32_t>(k >> 32));
            dmax = max(dmax, static_cast<uint32_t>(k >> 32));
          }
        }
        dmin = __reduce_min_sync(FULL, dmin);
        dmax = __reduce_max_sync(FULL, dmax);
        const uint32_t nbits = 32u - __clz(dmax - dmin);  // distance bits that differ (0..32)
#pragma unroll 1
        for (uint32_t j0 = 0; j0 < s; j0 += 32) {
          const uint32_t j = j0 + lane;
          if (j < s) {
            const uint64_t k = ck[j];
            const uint32_t hi = static_cast<uint32_t>(k >> 32) - dmin, lo = static_cast<uint32_t>(k);
            cd[j] = k == kMaxKey ? 0xFFFFFFFFu : (nbits >= 32 ? hi : __funnelshift_r(lo, hi, nbits));
          }
        }
      }
      if (s + lane < ((s + 3) & ~3u)) cd[s + lane] = 0xFFFFFFFFu;  // whole uint4 loads
      __syncwarp();
      bool clash = false;
#pragma unroll 1
      for (uint32_t j0 = 0; j0 < s; j0 += 32) {
        const uint32_t j = j0 + lane;
        const uint32_t d = j < s ? cd[j] : 0xFFFFFFFFu;
        uint32_t r = 0;
#pragma unroll 2
        for (uint32_t t = 0; t < s; t += 4) {
          const uint4 p4 = *reinterpret_cast<const uint4*>(cd + t);
          r += (p4.x < d ? 1u : 0u) + (p4.y < d ? 1u : 0u) + (p4.z < d ? 1u : 0u) + (p4.w < d ? 1u : 0u);
        }
        if (j < s && ck[j] != kMaxKey) {
          inv[r] = static_cast<uint8_t>(j);
          cke[j] = static_cast<uint8_t>(r);
        }
      }
      __syncwarp();
#pragma unroll 1
      for (uint32_t j0 = 0; j0 < s; j0 += 32) {
        const uint32_t j = j0 + lane;
        clash |= j < s && ck[j] != kMaxKey && inv[cke[j]] != j;
      }
      while (__any_sync(FULL, clash)) {  // rare: whole keys
        __syncwarp();
#pragma unroll 1
        for (uint32_t j0 = 0; j0 < s; j0 += 32) {
          const uint32_t j = j0 + lane;
          const uint64_t k = j < s ? ck[j] : kMaxKey;
          uint32_t r = 0, t = 0;
#pragma unroll 1
          for (; t + 2 <= s; t += 2) {
            const ulonglong2 p2 = *reinterpret_cast<const ulonglong2*>(ck + t);
            r += (p2.x < k ? 1u : 0u) + (p2.y < k ? 1u : 0u);
          }
          if (t < s) r += ck[t] < k ? 1u : 0u;
          if (k != kMaxKey) {
            GANN_CHECK(r < sreal);
            inv[r] = static_cast<uint8_t>(j);  // equal keys: one of them wins the slot
            cke[j] = static_cast<uint8_t>(r);
          }
        }
        __syncwarp();
        uint32_t lost = 0;
#pragma unroll 1
        for (uint32_t j0 = 0; j0 < s; j0 += 32) {
          const uint32_t j = j0 + lane;
          const bool loser = j < s && ck[j] != kMaxKey && inv[cke[j]] != j;
          lost += __popc(__ballot_sync(FULL, loser));
          if (loser) ck[j] = kMaxKey;
        }
        clash = lost != 0;
        sreal -= lost;
      }
      uint32_t p0 = 0xFFFFFFFFu, kept = 0;
#pragma unroll 1
      for (uint32_t j0 = 0; j0 < s; j0 += 32) {
        const uint32_t j = j0 + lane;
        bool in = false;
        if (j < s && ck[j] != kMaxKey) {
          p0 = min(p0, static_cast<uint32_t>(posb[j]));
          const uint32_t fin = posb[j] + cke[j];
          in = fin < L;
          if (in) atomicOr(bm + (fin >> 5), 1u << (fin & 31));
        }
        kept += __popc(__ballot_sync(FULL, in));
      }
      p0 = __reduce_min_sync(FULL, p0);
      nsurv += sreal;
      __syncwarp();
      // ---- rebuild positions [p0, new size), last chunk first (search_kernel's scheme) ----
      {
        constexpr int RB = GANN_SEARCH_RB;
        const uint32_t nsz = min(L, size + sreal);
        const int c_lo = static_cast<int>(p0 >> 5);
        uint32_t running = kept;
        int cb = static_cast<int>((nsz - 1) >> 5);
#pragma unroll 1
        for (; cb - c_lo + 1 >= RB; cb -= RB) {
          uint64_t key[RB];
          bool act[RB];
#pragma unroll
          for (int j = 0; j < RB; j++) {
            const int c = cb - j;
            const uint32_t wd = bm[c];
            running -= __popc(wd);
            const uint32_t t = static_cast<uint32_t>(c) * 32 + lane;
            const uint32_t before = running + __popc(wd & lanemask_lt(lane));
            act[j] = t >= p0 && t < nsz;
            const bool mine = (wd >> lane) & 1u;
            key[j] = 0;
            if (act[j]) {
              GANN_CHECK(t < L && (mine ? before < sreal : t - before < size));
              key[j] = mine ? ck[inv[before]] : beam[t - before];
            }
          }
          __syncwarp();
#pragma unroll
          for (int j = 0; j < RB; j++) {
            const int c = cb - j;
            if (act[j]) beam[static_cast<uint32_t>(c) * 32 + lane] = key[j];
            if (lane == 0) bm[c] = 0;
          }
        }
#pragma unroll 1
        for (; cb >= c_lo; cb--) {
          const uint32_t wd = bm[cb];
          running -= __popc(wd);
          const uint32_t t = static_cast<uint32_t>(cb) * 32 + lane;
          const uint32_t before = running + __popc(wd & lanemask_lt(lane));
          const bool act = t >= p0 && t < nsz;
          const bool mine = (wd >> lane) & 1u;
          uint64_t key = 0;
          if (act) {
            GANN_CHECK(t < L && (mine ? before < sreal : t - before < size));
            key = mine ? ck[inv[before]] : beam[t - before];
          }
          __syncwarp();
          if (act) beam[t] = key;
          if (lane == 0) bm[cb] = 0;
        }
      }
      size = min(L, size + sreal);
      hint = min(hint, p0);
      table_commit();
      __syncwarp();
    }

    __syncwarp();
    if (a.out_ids) {
#pragma unroll 1
      for (uint32_t i = lane; i < a.k_out; i += 32) {
        const bool have = i < size;
        a.out_ids[static_cast<uint64_t>(q) * a.k_out + i] = have ? bkey_id(beam[i]) : kNone;
        a.out_dists[static_cast<uint64_t>(q) * a.k_out + i] = have ? key_dist(beam[i]) : __int_as_float(0x7f800000);
      }
    }
    if (lane == 0) {
      if (a.n_visited) a.n_visited[q] = nvis;
      if (a.dist_comps) a.dist_comps[q] = evals;
      if (a.vis_ids && nvis > a.vcap) atomicAdd(a.overflow, 1u);
      if (a.stats) {
        atomicAdd(a.stats + kStQueries, 1ull);
        atomicAdd(a.stats + kStExpansions, static_cast<unsigned long long>(nvis));
        atomicAdd(a.stats + kStEvals, static_cast<unsigned long long>(evals));
        atomicAdd(a.stats + kStMerges, static_cast<unsigned long long>(steps));
        atomicAdd(a.stats + kStSurvivors, static_cast<unsigned long long>(nsurv));
        atomicAdd(a.stats + kStGuess, static_cast<unsigned long long>(dropped));
      }
    }
    __syncwarp();
    if (lane == 0) q = atomicAdd(a.next_query, 1u);
    q = __shfl_sync(FULL, q, 0);
  }
  // the region's next owner (any warp on the device) clears it before use: this
  // warp's last table stores must be visible device-wide before the release
  __threadfence();
  __syncwarp();
  if (lane == 0) atomicAnd(a.gtab_busy + g2_region / 32, ~(1u << (g2_region % 32)));
}

namespace {
template <int E, int M, int LPR, int CPL>
cudaError_t launch_batch(const SearchArgs& a, cudaStream_t s) {
  const uint32_t cm = a.batch_cm;
  uint32_t per_warp = static_cast<uint32_t>(search_batch_smem_per_warp(a.L, cm));
  if (const char* pv = std::getenv("GANN_BATCH_PAD")) per_warp += static_cast<uint32_t>(std::atoi(pv)) & ~15u;  // experiment
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e;
  const bool fit = a.stride == uint64_t(16) * LPR * CPL;
  auto k = fit ? search_batch_kernel<E, M, LPR, CPL, true> : search_batch_kernel<E, M, LPR, CPL, false>;
  if (a.nq == 0) return cudaSuccess;
  int sms = 0;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared)) !=
      cudaSuccess)
    return e;
  // CTA width (warps = queries per CTA; the kernel works per warp at any width)
  // and resident CTAs per SM. Shared memory and L1 share the SM's 256 KB, and
  // the rows a step gathers are in flight through L1 lines: with the carve-out
  // the resident CTAs' beams would take (6 CTAs of 4 warps at L = 832: 196 or
  // 228 KB) the 28-60 KB left for L1 throttle the gathers (measured at c1, L =
  // 832, 24 warps: 19.6 ms at 228 KB, 12.7 at 196, and 12.2 with 5 CTAs at 164
  // KB). So for each width the CTA count is lowered until L1 keeps ~4.5 KB per
  // resident warp, with the smallest carve-out that holds those CTAs; the
  // width with the most resident warps wins, on a tie the one that leaves more
  // L1, then the narrower one down to 2 warps (CTAs of a finishing launch free
  // their slots for the next launch sooner: 9.33 -> 9.02 ms per pipelined step
  // at L = 832; 1-warp CTAs pay the per-CTA kilobyte 4 times). GANN_BATCH_WPB / GANN_BATCH_CARVE
  // (percent) / GANN_BATCH_L1KB override (experiments).
  static const int kCarveKB[] = {8, 16, 32, 64, 100, 132, 164, 196, 228};
  uint32_t l1_per_warp = 4608;  // 4.5 KB
  if (const char* lv = std::getenv("GANN_BATCH_L1KB")) l1_per_warp = static_cast<uint32_t>(std::atoi(lv)) * 1024u;
  int forced_w = 0;
  if (const char* wv = std::getenv("GANN_BATCH_WPB")) forced_w = std::max(1, std::min(kWarpsPerBlock, std::atoi(wv)));
  int wpb = 0, per_sm = 0, pct = 100, best_carve = 0;
  for (int w = kWarpsPerBlock; w >= 1; w >>= 1) {
    if (size_t(per_warp) * w > static_cast<size_t>(optin)) continue;
    if (forced_w && w != forced_w && size_t(per_warp) * forced_w <= static_cast<size_t>(optin)) continue;
    int c = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k, w * 32, size_t(per_warp) * w)) != cudaSuccess) return e;
    c = std::max(1, c);
    const size_t cta = size_t(per_warp) * w + 1024;
    int carve = 228;
    for (; c >= 1; c--) {
      carve = 228;
      for (int kb : kCarveKB)
        if (size_t(kb) * 1024 >= cta * c) {
          carve = kb;
          break;
        }
      if (c == 1 || size_t(256 - carve) * 1024 >= size_t(c) * w * l1_per_warp) break;
    }
    // most resident warps; then most L1 left; then the narrower CTA (down to 2 warps)
    const bool better = c * w > per_sm * wpb ||
                        (c * w == per_sm * wpb && (carve < best_carve || (carve == best_carve && w >= 2)));
    if (wpb == 0 || better) {
      wpb = w;
      per_sm = c;
      best_carve = carve;
      pct = carve * 100 / 228;
    }
  }
  if (wpb == 0) return cudaErrorInvalidValue;  // the host checked the beam against the shared memory
  if (const char* cv = std::getenv("GANN_BATCH_CARVE")) {
    pct = std::atoi(cv);
    if ((e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, wpb * 32, size_t(per_warp) * wpb)) != cudaSuccess)
      return e;
  } else if ((e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct)) != cudaSuccess) {
    return e;
  }
  const size_t smem = size_t(per_warp) * wpb;
  const uint32_t want = (a.nq + wpb - 1) / wpb;
  const uint32_t blocks = std::min<uint32_t>(want, static_cast<uint32_t>(std::max(1, per_sm) * sms));
  if ((e = cudaMemsetAsync(a.next_query, 0, sizeof(uint32_t), s)) != cudaSuccess) return e;
  if (const char* dv = std::getenv("GANN_BATCH_DEBUG"))
    if (*dv == '1') std::fprintf(stderr, "batch launch: L %u cm %u per_warp %u wpb %d per_sm %d blocks %u\n", a.L, cm, per_warp, wpb, per_sm, blocks);
  k<<<blocks, wpb * 32, smem, s>>>(a, per_warp, cm);
  return cudaGetLastError();
}
}  // namespace

}  // namespace gann
