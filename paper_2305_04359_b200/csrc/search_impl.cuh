// search.cu — batched greedy beam search, one warp per query (sm_100a).
//
// Behaviour contract: graphann::beam_search (src/search.cpp:62-131), restated
// in SURVEY.md §B.1. Per warp:
//   * the beam (<= L keys, sorted) and its expanded flags live in shared
//     memory; a merge moves only the tail behind the first insertion point,
//     in place, last 32-entry chunk first (targets only move right);
//   * exactly one vertex is expanded per step (the first unexpanded key,
//     src/search.cpp:96-103), gated by the k-th best key with epsilon slack
//     (:105-107) — the only order the reference's visit sequence allows;
//   * the expanded vertex's adjacency row (R ids, one coalesced load) is run
//     through the visited filter, the surviving ids' rows are gathered with
//     16-byte loads (LPR lanes per row, several rows in flight per lane) and
//     reduced with xor-shuffles into exact int32 (u8/i8) or f32 distances;
//   * the new keys are merged into the beam as top-L of the union with exact
//     (dist, id) duplicates dropped — equal to the reference's sequential
//     push (:83-90) because the L-th key only ever decreases.
// Visited filter. FAST: a direct-mapped table in shared memory that
// overwrites on collision (one load + one store per neighbour; it keeps the
// most recent ids, which is what graph locality re-encounters). An evicted id
// may be evaluated again, but the table never reports a false positive, so
// ids / |V| / visit order are the reference's; re-evaluated
// keys that are still in the beam are dropped as exact duplicates. REF: the reference's own ApproxVisitedSet
// (L*L slots, mix64(id ^ seed) % L^2, include/graphann/search.hpp:24-38,
// seed from src/search.cpp:52-58) in global memory, applied per expansion
// with the order-exact warp rule of SURVEY.md §0.4 (first lane of a slot
// tests, last lane writes), so dist_comps matches the reference too. EXACT:
// an open-addressing set per query in global memory that never forgets, so
// dist_comps is the number of distinct ids evaluated (U in SURVEY.md §8d);
// used to account the algorithmic bytes of a launch.
#pragma once
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace gann {

namespace {

constexpr int kWarpsPerBlock = kSearchWarpsPerBlock;
#ifndef GANN_SEARCH_MINB
#define GANN_SEARCH_MINB 6  // resident CTAs per SM the register budget targets (80 regs; 7 CTAs at 72 regs
                            // rematerialised more and measured 1.2% slower)
#endif
#ifndef GANN_SEARCH_MINB_WIDE
#define GANN_SEARCH_MINB_WIDE 7  // rows of 16 lanes (256-byte u8 rows): left free the compiler takes 76
                                 // registers, 6 CTAs, and c2 ran 7% slower than at 7 CTAs
#endif

#ifndef GANN_SEARCH_MINB_G2
#define GANN_SEARCH_MINB_G2 6  // large beams, rows <= 256 B: 7 (72 registers; shared memory allows 7 CTAs) measured
                               // 33% slower at c1 L=832 (19.8 vs 14.8 ms)
#endif

// Rows in flight per lane group per pass: U <= LPR so the transposed
// reduction can hand every lane of the group (at most) one finished row.
#ifndef GANN_SEARCH_RB
#define GANN_SEARCH_RB 4  // beam chunks rebuilt per batch after a merge (see the loop)
#endif
#ifndef GANN_SEARCH_U
#define GANN_SEARCH_U 8  // rows in flight per lane group (registers: U * CPL * 4)
#endif
template <int LPR, int CPL>
struct Unroll {
  static constexpr int raw = LPR > GANN_SEARCH_U ? GANN_SEARCH_U : LPR;
  static constexpr int U = (raw / CPL) < 1 ? 1 : (raw / CPL);
};

// Beam keys: (order-preserving f32 dist) << 32 | id << 1 | expanded. The flag
// is the least significant bit, so key order is still (dist, id) order
// (neighbor_less) and a u64 compare needs no mask; ids are below 2^31 (the
// host checks n). The flag bit replaced a byte array of L flags per warp:
// less shared memory per query and no flag copy in the tail rebuild.
__device__ __forceinline__ uint64_t make_bkey(float d, uint32_t id) {
  return (static_cast<uint64_t>(f2ord(d)) << 32) | (static_cast<uint64_t>(id) << 1);
}
__device__ __forceinline__ uint32_t bkey_id(uint64_t k) { return static_cast<uint32_t>(k) >> 1; }

// Chunk `base` of row `id`: one IMAD.WIDE.U32 (id * stride + the 64-bit
// per-lane chunk base); the compiler's own lowering of size_t(id) * stride +
// base took three instructions per row.
__device__ __forceinline__ const uint4* row_chunk(const uint8_t* base, uint32_t id, uint32_t stride) {
  uint64_t p;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(id), "r"(stride), "l"(reinterpret_cast<uint64_t>(base)));
  return reinterpret_cast<const uint4*>(p);
}

// One pass: lane group g (LPR lanes) takes UU consecutive rows from b0 + g*UU,
// their ids from one vectorised shared load. FIT: the row is exactly LPR*CPL
// chunks (d = 128 u8 at 8 lanes), so no chunk is predicated off.
template <class Op, int LPR, int CPL, int UU, bool FIT>
__device__ __forceinline__ void eval_pass(uint32_t b0, const uint32_t* ids, uint32_t m, uint32_t stride,
                                          const uint8_t* const (&cb)[CPL], const bool (&chv)[CPL],
                                          uint64_t* out, const uint4 (&qr)[CPL], int sub, int grp,
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
    for (int c = 0; c < CPL; c++)
      x[u][c] = __ldg(row_chunk(cb[c], id[u], stride));
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
  // keys below the L-th beam key are appended to out (candidate order is not
  // needed: the merge ranks them)
  uint64_t key = kMaxKey;
  if (sub < UU && r < m) key = make_bkey(Op::finish(tot), ids[r]);
  const bool keep = key < worst;
  const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
  GANN_CHECK(!keep || n_out + __popc(bal & ((1u << lane) - 1u)) < m);
  if (keep) out[n_out + __popc(bal & ((1u << lane) - 1u))] = key;
  n_out += __popc(bal);
}

// Distances from the lane's query chunks qr to rows ids[0..m); the keys below
// `worst` go to out[0..returned count).
// Full passes take RPP*U rows; the last, partial pass shrinks to a quarter or
// half of that when the remaining rows fit (fewer instructions for the same
// rows). ids[] must be padded with valid vertex ids up to the next multiple of
// RPP*U (<= 32): passes load whole without per-row predicates, and each row
// address is one IMAD.WIDE.U32 (id * stride + the lane's hoisted chunk base).
// A chunk index beyond the row (nch not a multiple of LPR) is clamped to the
// row's last chunk and its contribution predicated off.
template <class Op, int LPR, int CPL, bool FIT>
__device__ __forceinline__ uint32_t eval_rows(const uint8_t* __restrict__ data, uint32_t stride,
                                              uint32_t nch, const uint32_t* ids, uint32_t m,
                                              uint64_t* out, const uint4 (&qr)[CPL], int lane,
                                              uint64_t worst) {
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
    eval_pass<Op, LPR, CPL, U, FIT>(b0, ids, m, stride, cb, chv, out, qr, sub, grp, worst, n_out, lane);
  const uint32_t rem = m - b0;
  if (rem == 0) return n_out;
  if (U >= 8 && rem <= RPP * (U / 4))
    eval_pass<Op, LPR, CPL, (U >= 8 ? U / 4 : 1), FIT>(b0, ids, m, stride, cb, chv, out, qr, sub, grp, worst, n_out, lane);
  else if (U >= 4 && rem <= RPP * (U / 2))
    eval_pass<Op, LPR, CPL, (U >= 4 ? U / 2 : 1), FIT>(b0, ids, m, stride, cb, chv, out, qr, sub, grp, worst, n_out, lane);
  else
    eval_pass<Op, LPR, CPL, U, FIT>(b0, ids, m, stride, cb, chv, out, qr, sub, grp, worst, n_out, lane);
  return n_out;
}

__device__ __forceinline__ uint32_t lanemask_lt(int lane) { return (1u << lane) - 1u; }

}  // namespace

size_t search_smem_per_warp(uint32_t L, uint32_t R, uint32_t hash_log2, bool hash16);

// F16: the fast mode with u16 slots, compiled without the other modes'
// branches and without the diagnostic counters (filter drops, adjacency
// entries, merges, survivors, moved, duplicates); the general instance keeps
// them (GANN_SEARCH_DIAG=1 selects it for the fast mode too)
// R64: the degree bound is 64 (every BASELINE config), fixed at compile time
// FIT: rows are exactly LPR * CPL chunks (no chunk predicate in the gather)
// G2: the second-level visited table (large beams; its own instance so the
// registers it takes, 72 -> 79, do not cost the small beams a resident CTA)
template <int E, int M, int LPR, int CPL, bool F16, bool R64 = false, bool FIT = false, bool G2 = false>
__global__ void __launch_bounds__(kWarpsPerBlock * 32,
                                  G2 && LPR * CPL <= 16 ? GANN_SEARCH_MINB_G2 : (LPR >= 16 ? GANN_SEARCH_MINB_WIDE : GANN_SEARCH_MINB))
    search_kernel(const SearchArgs a, const uint32_t per_warp) {
  using Op = DistOp<E, M>;
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint32_t L = a.L, R = R64 ? 64u : a.R;
  const uint32_t Lp = (L + 31) & ~31u, Rp = (R + 31) & ~31u;
  const uint32_t hlog2 = a.hash_log2;
  const uint32_t H = 1u << hlog2;
  const uint32_t nch = static_cast<uint32_t>(a.stride >> 4);
  const uint32_t stride32 = static_cast<uint32_t>(a.stride);  // host: stride < 2^32
  uint8_t* base = smem + wib * per_warp;
  uint64_t* beam = reinterpret_cast<uint64_t*>(base);
  // ck: candidate keys; tmpk: keys below the L-th (dead after the duplicate
  // pass, so it also holds the sorted survivors srt); cid: candidate ids
  // (dead after the gather, so it also holds the insertion points posb)
  uint64_t* ck = beam + Lp;
  uint64_t* tmpk = ck + Rp;
  uint64_t* srt = tmpk;
  uint32_t* cid = reinterpret_cast<uint32_t*>(tmpk + Rp);
  uint32_t* posb = cid;
  uint32_t* hash = cid + Rp;
  uint16_t* h16 = reinterpret_cast<uint16_t*>(hash);
  const uint32_t hbits = a.hash_bits;  // F16 implies hbits != 0
  const int vmode = F16 ? 0 : a.visited_mode;
  const uint32_t hmask = hbits ? (1u << hbits) - 1u : 0u;
  uint32_t* bm = hash + (hbits ? H / 2 : H);  // Lp bits: final positions of a merge's survivors
  // (no flag array: a beam key's lowest bit is its expanded flag, make_bkey)
  const uint32_t FULL = 0xFFFFFFFFu;

  // Second-level visited table (large beams, fast mode): the ids the shared
  // table has forgotten are looked up in a 16k-slot table of this warp's own
  // region in global memory before their rows are gathered again (c1, L = 832:
  // 40.8k evaluations per query with the 1024-slot shared table against 9.1k
  // distinct ids). Exact-positive like the shared table (u16 remainders of a
  // bijective hash, n <= 2^27), so results do not depend on it.
  uint64_t* g2 = nullptr;
  uint32_t g2_region = kNone;
  // L2 policy of the second-level table's accesses: evict_last keeps the
  // resident warps' regions in L2 against the stream of gathered rows
  // (GANN_GTAB_KEEP=0: evict_normal)
  uint64_t g2pol = 0;
  if (G2) {
    if (a.gtab_keep)
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(g2pol));
    else
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(g2pol));
  }
  if (G2 && F16 && a.gtab && a.n <= (1u << (a.gtab_log2 + 15))) {
    if (lane == 0) {
      const uint32_t words = (a.gtab_regions + 31) / 32;
      uint32_t w0 = (blockIdx.x * 32 + (threadIdx.x >> 5)) % words;
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
    if (g2_region != kNone) g2 = a.gtab + (static_cast<uint64_t>(g2_region) << a.gtab_log2);
  }
  const uint32_t g2mask = (1u << (a.gtab_log2 + 15)) - 1u;

  // Persistent warps: a resident grid pulls queries from a global counter, so
  // slow queries do not leave whole CTAs idle at the end of a wave.
  uint32_t q = 0;
  if (lane == 0) q = atomicAdd(a.next_query, 1u);
  q = __shfl_sync(0xFFFFFFFFu, q, 0);
  for (; q < a.nq;) {
    if (G2 && g2) {  // an empty table for this query (0xFFFF: no remainder)
      for (uint32_t i = lane; i < (1u << a.gtab_log2) / 2; i += 32)
        asm volatile("st.global.cg.L2::cache_hint.v4.u32 [%0], {%1, %1, %1, %1}, %2;"
                     :: "l"(reinterpret_cast<uint4*>(g2) + i), "r"(kNone), "l"(g2pol) : "memory");
    }
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
    uint32_t* table = nullptr;
    uint64_t seed = 0;
    const uint32_t LL = L * L;
    const uint32_t TS = a.exact_slots;  // mode 2: exact open-addressing set, global memory
    if (vmode == 2) {
      table = a.ref_table + static_cast<uint64_t>(q) * TS;
      for (uint32_t i = lane; i < TS; i += 32) table[i] = kNone;
    } else if (vmode == 1) {
      table = a.ref_table + static_cast<uint64_t>(q) * LL;
      for (uint32_t i = lane; i < LL; i += 32) table[i] = kNone;
      // search_seed — src/search.cpp:52-58 (rows are zero padded to >= 16 bytes,
      // which equals the reference's zero-filled copy of the first min(16, bytes))
      const uint64_t* q64 = reinterpret_cast<const uint64_t*>(qp);
      const uint64_t h = mix64(start, a.dim);
      seed = mix64(h ^ q64[0], q64[1]);
    } else {
      for (uint32_t i = lane; i < (hbits ? H / 2 : H); i += 32) hash[i] = kNone;  // u16 slots: 0xFFFF
    }
    for (uint32_t i = lane; i < Lp / 32; i += 32) bm[i] = 0;
    cid[lane] = start;  // padded: eval_rows loads whole passes
    __syncwarp();
    eval_rows<Op, LPR, CPL, FIT>(a.data, stride32, nch, cid, 1, ck, qr, lane, kMaxKey);
    __syncwarp();
    if (lane == 0) {
      beam[0] = ck[0];
      if (vmode == 2)
        table[(start * 0x9E3779B1u) & (TS - 1)] = start;
      else if (vmode == 1)
        table[mix64(static_cast<uint64_t>(start) ^ seed) % LL] = start;
      else if (G2 && a.hash_log2 == 0) {
        // no shared table (the second level alone): nothing to enter
      } else if ((F16 || hbits) && a.hash_ways == 4) {
        const uint32_t h = (start * 0x9E3779B1u) & hmask;
        reinterpret_cast<uint64_t*>(hash)[h >> 15] = 0xFFFFFFFFFFFF0000ull | (h & 0x7FFFu);
      } else if ((F16 || hbits) && a.hash_ways == 2) {
        const uint32_t h = (start * 0x9E3779B1u) & hmask;
        hash[h >> 15] = 0xFFFF0000u | (h & 0x7FFFu);
      } else if (F16 || hbits) {
        const uint32_t h = (start * 0x9E3779B1u) & hmask;
        h16[h >> 15] = static_cast<uint16_t>(h & 0x7FFFu);
      } else if (a.hash_ways == 4) {
        reinterpret_cast<uint4*>(hash)[(start * 0x9E3779B1u) >> (34 - hlog2)] = make_uint4(start, kNone, kNone, kNone);
      } else
        hash[(start * 0x9E3779B1u) >> (32 - hlog2)] = start;
    }
    uint32_t size = 1, nvis = 0, hint = 0, evict = 0;
    uint64_t evals = 1;
    uint32_t adjsum = 0, merges = 0, survivors = 0, moved = 0, dups = 0, ghits = 0;  // per query: 32 bits suffice
    // speculative register prefetch of the next expansion's adjacency row
    // (R <= 64: two ids per lane); used when the guess turns out right
    const bool pf_ok = R <= 64;
    uint32_t pf_id = kNone, pf0 = kNone, pf1 = kNone;
    uint64_t pf_key = kMaxKey;  // the guess's beam key (large beams)
    // second-level table words of the guess's neighbours, read behind this
    // step's gather so the next step's filter does not wait on L2 (pw_id: the
    // vertex they belong to)
    uint64_t pw0 = 0, pw1 = 0;
    uint32_t pw_id = kNone;
    // the guess's second-level words (its row has arrived by the time this
    // runs: behind a gather, or it is waited for)
    auto g2_prefetch = [&]() {
      if (G2 && g2 && pf_id != kNone && pw_id != pf_id) {
        const uint32_t b0 = ((pf0 * 0x85EBCA6Bu) & g2mask) >> 15, b1 = ((pf1 * 0x85EBCA6Bu) & g2mask) >> 15;
        pw0 = 0ull;
        pw1 = 0ull;
        if (pf0 != kNone)
          asm volatile("ld.global.cg.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(pw0) : "l"(g2 + b0), "l"(g2pol) : "memory");
        if (pf1 != kNone)
          asm volatile("ld.global.cg.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(pw1) : "l"(g2 + b1), "l"(g2pol) : "memory");
        pw_id = pf_id;
      }
    };
    __syncwarp();

    while (true) {
      // first unexpanded key at or after `hint` (everything before is expanded)
      int fu = -1;
      uint32_t fbal = 0, fb0 = 0;
      for (uint32_t b0 = hint & ~31u; b0 < size; b0 += 32) {
        const uint32_t i = b0 + lane;
        const uint32_t bal = __ballot_sync(FULL, i >= hint && i < size && (beam[i] & 1ull) == 0);
        if (bal) {
          fu = static_cast<int>(b0 + __ffs(bal) - 1);
          fbal = bal;
          fb0 = b0;
          break;
        }
      }
      if (fu < 0) break;
      const uint64_t fk = beam[fu];
      if (a.k_gate <= size) {  // k-gate + epsilon, src/search.cpp:105-107
        const float bk = key_dist(beam[a.k_gate - 1]);
        const float lim = __fadd_rn(bk, __fmul_rn(a.eps, fabsf(bk)));
        if (key_dist(fk) > lim) break;
      }
      const uint32_t cur = bkey_id(fk);
      hint = fu + 1;
      const uint32_t* row = graph_row(a.graph, cur, R);
      uint32_t nb0 = kNone, nb1 = kNone;
      bool use_pw = false;
      if (pf_ok) {
        if (pf_id == cur) {
          nb0 = pf0;
          nb1 = pf1;
          if (!F16) ghits++;
          use_pw = G2 && g2 && pw_id == cur;
        } else {
          nb0 = lane < R ? __ldg(row + lane) : kNone;
          nb1 = lane + 32 < R ? __ldg(row + 32 + lane) : kNone;
        }
        // guess the next expansion: the next unexpanded key after fu
        const uint32_t above = fbal & ~((2u << (fu - fb0)) - 1u);
        int gi = above ? static_cast<int>(fb0 + __ffs(above) - 1) : -1;
        if (gi < 0 && fb0 + 32 < size) {
          const uint32_t i = fb0 + 32 + lane;
          const uint32_t bal = __ballot_sync(FULL, i < size && (beam[i] & 1ull) == 0);
          if (bal) gi = static_cast<int>(fb0 + 32 + __ffs(bal) - 1);
        }
        const uint64_t gk = gi >= 0 ? beam[gi] : kMaxKey;
        if (G2) pf_key = gk;
        pf_id = gi >= 0 ? bkey_id(gk) : kNone;
        if (pf_id != kNone) {
          const uint32_t* prow = graph_row(a.graph, pf_id, R);
          pf0 = lane < R ? __ldg(prow + lane) : kNone;
          pf1 = lane + 32 < R ? __ldg(prow + 32 + lane) : kNone;
        }
      }
      __syncwarp();
      if (lane == 0) {
        beam[fu] = fk | 1ull;  // expanded
        if (a.vis_ids && nvis < a.vcap) {
          a.vis_ids[static_cast<uint64_t>(q) * a.vcap + nvis] = cur;
          a.vis_dists[static_cast<uint64_t>(q) * a.vcap + nvis] = key_dist(fk);
        }
      }
      nvis++;

      // ---- neighbours through the visited filter (adjacency order kept) ----
      uint32_t m = 0;
      for (uint32_t t0 = 0; t0 < R; t0 += 32) {
        const uint32_t t = t0 + lane;
        const uint32_t nb = pf_ok ? (t0 == 0 ? nb0 : nb1) : (t < R ? __ldg(row + t) : kNone);
        const bool valid = nb != kNone;
        if (!F16) adjsum += __popc(__ballot_sync(FULL, valid));
        bool fresh;
        if (vmode == 2) {
          fresh = false;
          if (valid) {
            uint32_t slot = (nb * 0x9E3779B1u) & (TS - 1);
            while (true) {
              const uint32_t old = atomicCAS(table + slot, kNone, nb);
              if (old == kNone) { fresh = true; break; }
              if (old == nb) break;
              slot = (slot + 1) & (TS - 1);
            }
          }
        } else if (vmode == 1) {
          const uint32_t slot =
              valid ? static_cast<uint32_t>(mix64(static_cast<uint64_t>(nb) ^ seed) % LL) : kNone;
          const uint32_t peers = __match_any_sync(FULL, slot);
          const bool first = (__ffs(peers) - 1) == lane;
          const bool last = (31 - __clz(peers)) == lane;
          const uint32_t tv = valid ? table[slot] : 0u;
          const bool seen = valid && first && tv == nb;
          __syncwarp();
          if (valid && last) table[slot] = nb;
          __syncwarp();
          fresh = valid && !seen;
        } else if (G2 && a.hash_log2 == 0) {
          fresh = valid;  // no shared table: the second level alone decides
        } else if ((F16 || hbits) && a.hash_ways == 4) {
          // 4-way buckets of u16 slots in one u64 (newest in the low half
          // word), as the 2-way case below
          const uint32_t h = (nb * 0x9E3779B1u) & hmask;
          const uint32_t bucket = h >> 15, rem = h & 0x7FFFu;
          uint64_t* h64 = reinterpret_cast<uint64_t*>(hash);
          const uint64_t w = valid ? h64[bucket] : 0ull;
          const uint32_t rr = rem | (rem << 16);
          const uint32_t eq = __vcmpeq2(static_cast<uint32_t>(w), rr) | __vcmpeq2(static_cast<uint32_t>(w >> 32), rr);
          fresh = valid && eq == 0u;
          __syncwarp();
          if (fresh) {
            h64[bucket] = (w << 16) | rem;
            if (!F16) evict += (w >> 48) != 0xFFFFu ? 1u : 0u;
          }
        } else if ((F16 || hbits) && a.hash_ways == 2) {
          // 2-way buckets of u16 slots (word = older << 16 | newer): bucket and
          // remainder of a bijection of the id over hbits bits, so a match is
          // the same id; 0xFFFF (no 15-bit remainder) marks an empty slot. An
          // insert shifts the newer slot up and evicts the older id.
          const uint32_t h = (nb * 0x9E3779B1u) & hmask;
          const uint32_t bucket = h >> 15, rem = h & 0x7FFFu;
          const uint32_t w = valid ? hash[bucket] : 0u;
          fresh = valid && (w & 0xFFFFu) != rem && (w >> 16) != rem;
          __syncwarp();
          if (fresh) {
            hash[bucket] = (w << 16) | rem;
            if (!F16) evict += (w >> 16) != 0xFFFFu ? 1u : 0u;
          }
        } else if (F16 || hbits) {
          // direct-mapped u16 slots: slot and remainder of a bijection of the
          // id over hbits bits (id < 2^hbits), so a match is the same id;
          // 0xFFFF (no 15-bit remainder) marks an empty slot
          const uint32_t h = (nb * 0x9E3779B1u) & hmask;
          const uint32_t slot = h >> 15, rem = h & 0x7FFFu;
          const uint32_t old = valid ? h16[slot] : 0xFFFFu;
          fresh = valid && old != rem;
          __syncwarp();
          if (fresh) {
            h16[slot] = static_cast<uint16_t>(rem);
            if (!F16) evict += old != 0xFFFFu ? 1u : 0u;
          }
        } else if (a.hash_ways == 4) {
          // ids too wide for u16 remainders (n > 2^26): 4-way buckets of u32
          // ids, one 16-byte load; an insert shifts the bucket, dropping its
          // oldest id
          uint4* h4 = reinterpret_cast<uint4*>(hash);
          const uint32_t bucket = (nb * 0x9E3779B1u) >> (34 - hlog2);
          const uint4 w = valid ? h4[bucket] : make_uint4(kNone, kNone, kNone, kNone);
          fresh = valid && w.x != nb && w.y != nb && w.z != nb && w.w != nb;
          __syncwarp();
          if (fresh) {
            h4[bucket] = make_uint4(nb, w.x, w.y, w.z);
            evict += w.w != kNone ? 1u : 0u;
          }
        } else {
          // direct-mapped, overwrite on collision: never a false positive
          const uint32_t slot = (nb * 0x9E3779B1u) >> (32 - hlog2);
          const uint32_t old = valid ? hash[slot] : kNone;
          fresh = valid && old != nb;
          __syncwarp();
          if (fresh) {
            hash[slot] = nb;
            evict += old != kNone ? 1u : 0u;
          }
        }
        if (G2 && F16 && g2 && __any_sync(FULL, fresh)) {
          // not in the shared table: the second level decides (and learns it)
          const uint32_t h = (nb * 0x85EBCA6Bu) & g2mask;
          const uint32_t bucket = h >> 15, rem = h & 0x7FFFu;
          uint64_t w = 0ull;
          if (use_pw)
            w = t0 == 0 ? pw0 : pw1;  // read behind the previous step's gather (no insert since)
          else if (fresh)
            asm volatile("ld.global.cg.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(w) : "l"(g2 + bucket), "l"(g2pol) : "memory");
          const uint32_t rr = rem | (rem << 16);
          if (fresh && (__vcmpeq2(static_cast<uint32_t>(w), rr) | __vcmpeq2(static_cast<uint32_t>(w >> 32), rr)))
            fresh = false;
          else if (fresh)
            asm volatile("st.global.cg.L2::cache_hint.u64 [%0], %1, %2;" :: "l"(g2 + bucket), "l"((w << 16) | rem), "l"(g2pol) : "memory");
        }
        const uint32_t bal = __ballot_sync(FULL, fresh);
        GANN_CHECK(!fresh || m + __popc(bal & lanemask_lt(lane)) < Rp);
        if (fresh) cid[m + __popc(bal & lanemask_lt(lane))] = nb;
        m += __popc(bal);
      }
      pw_id = kNone;  // this step's inserts made any earlier read stale
      if (m == 0) {
        if (G2 && a.next_pf) g2_prefetch();
        continue;
      }
      GANN_CHECK(((m + 31) & ~31u) <= Rp);
      if (m + lane < ((m + 31) & ~31u)) cid[m + lane] = cur;  // pad to a whole pass
      __syncwarp();
      evals += m;
      // distances; keys below the L-th beam key go to tmpk (c1 of them)
      const uint64_t worst = size == L ? beam[L - 1] : kMaxKey;
      const uint32_t c1 = eval_rows<Op, LPR, CPL, FIT>(a.data, stride32, nch, cid, m, tmpk, qr, lane, worst);
      if (G2 && a.next_pf) g2_prefetch();
      if (c1 == 0) continue;
      __syncwarp();
      // ---- merge: top-L of beam U new, exact duplicates dropped ----
      // insertion points; exact (dist, id) duplicates of beam keys drop
      uint32_t s = 0;
      uint64_t mk = kMaxKey;  // the smallest survivor (large beams)
      for (uint32_t j0 = 0; j0 < c1; j0 += 32) {
        const uint32_t j = j0 + lane;
        bool keep = j < c1;
        const uint64_t k = keep ? tmpk[j] : kMaxKey;
        uint32_t pb = 0;
        if (keep) {
          pb = lower_bound_steps_u64(beam, size, k);
          if (pb < size && (beam[pb] | 1ull) == (k | 1ull)) {  // the same (dist, id), expanded or not
            keep = false;
            if (!F16) dups++;
          }
        }
        const uint32_t bal = __ballot_sync(FULL, keep);
        if (G2 && keep) mk = min(mk, k);
        if (keep) {
          const uint32_t o = s + __popc(bal & lanemask_lt(lane));
          GANN_CHECK(o < Rp && pb <= size);
          ck[o] = k;
          posb[o] = pb;
        }
        s += __popc(bal);
      }
      if (s == 0) continue;
      if (G2 && pf_ok && a.next_pf) {
        // The next expansion is known before the rest of the merge: the
        // smaller of the guess (the first unexpanded key after fu) and the
        // smallest survivor. When a survivor beats the guess its row is
        // loaded now, behind the merge, instead of at the top of the next
        // step (which still checks pf_id == cur before using it). Survivors,
        // not new keys: re-evaluated beam keys (the filter forgets) would
        // point it at expanded vertices.
        const uint32_t mh = __reduce_min_sync(FULL, static_cast<uint32_t>(mk >> 32));
        const uint32_t ml =
            __reduce_min_sync(FULL, static_cast<uint32_t>(mk >> 32) == mh ? static_cast<uint32_t>(mk) : kNone);
        mk = (static_cast<uint64_t>(mh) << 32) | ml;
        if (mk < pf_key) {
          pf_key = mk;
          pf_id = bkey_id(mk);
          const uint32_t* prow = graph_row(a.graph, pf_id, R);
          pf0 = lane < R ? __ldg(prow + lane) : kNone;
          pf1 = lane + 32 < R ? __ldg(prow + 32 + lane) : kNone;
        }
      }
      __syncwarp();
      // survivors sorted (srt), final positions fin = insertion point + rank
      // marked in a bitmap of beam positions (only fin < L is kept)
      uint32_t p0 = 0xFFFFFFFFu, kept = 0;
      for (uint32_t j0 = 0; j0 < s; j0 += 32) {
        const uint32_t j = j0 + lane;
        bool in = false;
        if (j < s) {
          const uint64_t k = ck[j];
          // rank among the survivors (ck is 16-byte aligned: two keys per load)
          uint32_t r = 0, t = 0;
          for (; t + 2 <= s; t += 2) {
            const ulonglong2 p2 = *reinterpret_cast<const ulonglong2*>(ck + t);
            r += (p2.x < k ? 1u : 0u) + (p2.y < k ? 1u : 0u);
          }
          if (t < s) r += ck[t] < k ? 1u : 0u;
          GANN_CHECK(r < s);
          srt[r] = k;
          p0 = min(p0, posb[j]);
          const uint32_t fin = posb[j] + r;
          in = fin < L;
          if (in) atomicOr(bm + (fin >> 5), 1u << (fin & 31));
        }
        kept += __popc(__ballot_sync(FULL, in));
      }
      p0 = __reduce_min_sync(FULL, p0);
      if (!F16) {
        merges++;
        survivors += s;
        moved += size - p0;
      }
      __syncwarp();
      // rebuild positions [p0, new size) chunk by chunk, last chunk first:
      // position t holds survivor #before(t) if its bit is set, else the old
      // entry t - before(t); sources never lie above t, so descending chunks
      // read only entries not yet overwritten
      //
      // GANN_SEARCH_RB chunks at a time: their sources are all read (independent
      // loads in flight together) before any of them is written — sources lie
      // at or below their target, so a batch only reads entries of its own
      // chunks or lower ones, none written yet (one chunk at a time is a chain
      // of dependent shared-memory round trips: -2.7% at c1, L = 832). The
      // low remainder goes one chunk at a time (small beams rebuild 1-3
      // chunks: whole batches there cost the build's L = 128 searches 12%).
      {
        constexpr int RB = GANN_SEARCH_RB;
        const uint32_t nsz = min(L, size + s);
        const int c_lo = static_cast<int>(p0 >> 5);
        uint32_t running = kept;
        int cb = static_cast<int>((nsz - 1) >> 5);
        for (; cb - c_lo + 1 >= RB; cb -= RB) {  // whole batches from the top
          uint64_t key[RB];
          bool act[RB];
#pragma unroll
          for (int j = 0; j < RB; j++) {
            const int c = cb - j;
            const uint32_t w = bm[c];
            running -= __popc(w);
            const uint32_t t = static_cast<uint32_t>(c) * 32 + lane;
            const uint32_t before = running + __popc(w & lanemask_lt(lane));
            act[j] = t >= p0 && t < nsz;
            // one load from either source (no divergent branch)
            const bool mine = (w >> lane) & 1u;
            const uint64_t* src = mine ? srt + before : beam + (t - before);
            key[j] = 0;
            if (act[j]) {
              GANN_CHECK(t < L && (mine ? before < s : t - before < size));
              key[j] = *src;  // (a survivor's flag bit is 0: unexpanded)
            }
          }
          __syncwarp();  // every read of these chunks' old entries precedes their writes
#pragma unroll
          for (int j = 0; j < RB; j++) {
            const int c = cb - j;
            if (act[j]) beam[static_cast<uint32_t>(c) * 32 + lane] = key[j];
            if (lane == 0) bm[c] = 0;
          }
          // no second sync: the next (lower) batch reads only positions below
          // these chunks, none written yet
        }
        for (; cb >= c_lo; cb--) {  // the rest (small beams: usually all of it) one chunk at a time
          const uint32_t w = bm[cb];
          running -= __popc(w);
          const uint32_t t = static_cast<uint32_t>(cb) * 32 + lane;
          const uint32_t before = running + __popc(w & lanemask_lt(lane));
          const bool act = t >= p0 && t < nsz;
          const bool mine = (w >> lane) & 1u;
          const uint64_t* src = mine ? srt + before : beam + (t - before);
          uint64_t key = 0;
          if (act) {
            GANN_CHECK(t < L && (mine ? before < s : t - before < size));
            key = *src;
          }
          __syncwarp();
          if (act) beam[t] = key;
          if (lane == 0) bm[cb] = 0;
        }
      }
      size = min(L, size + s);
      hint = min(hint, p0);
      __syncwarp();
    }

    __syncwarp();
    // neighbors = top-k of V == beam prefix (every key above the first
    // unexpanded one has been expanded; k_out <= k_gate is enforced by the host)
    if (a.out_ids) {
      for (uint32_t i = lane; i < a.k_out; i += 32) {
        const bool have = i < size;
        a.out_ids[static_cast<uint64_t>(q) * a.k_out + i] = have ? bkey_id(beam[i]) : kNone;
        a.out_dists[static_cast<uint64_t>(q) * a.k_out + i] =
            have ? key_dist(beam[i]) : __int_as_float(0x7f800000);
      }
    }
    evict = __reduce_add_sync(FULL, evict);
    dups = __reduce_add_sync(FULL, dups);
    if (lane == 0) {
      if (a.n_visited) a.n_visited[q] = nvis;
      if (a.dist_comps) a.dist_comps[q] = evals;
      if (a.vis_ids && nvis > a.vcap) atomicAdd(a.overflow, 1u);
      if (a.stats) {
        atomicAdd(a.stats + kStQueries, 1ull);
        atomicAdd(a.stats + kStExpansions, static_cast<unsigned long long>(nvis));
        atomicAdd(a.stats + kStEvals, static_cast<unsigned long long>(evals));
        if (!F16) {
          atomicAdd(a.stats + kStDrops, static_cast<unsigned long long>(evict));
          atomicAdd(a.stats + kStAdj, static_cast<unsigned long long>(adjsum));
          atomicAdd(a.stats + kStMerges, static_cast<unsigned long long>(merges));
          atomicAdd(a.stats + kStSurvivors, static_cast<unsigned long long>(survivors));
          atomicAdd(a.stats + kStMoved, static_cast<unsigned long long>(moved));
          atomicAdd(a.stats + kStDups, static_cast<unsigned long long>(dups));
          atomicAdd(a.stats + kStGuess, static_cast<unsigned long long>(ghits));
        }
      }
    }
    __syncwarp();
    if (lane == 0) q = atomicAdd(a.next_query, 1u);
    q = __shfl_sync(0xFFFFFFFFu, q, 0);
  }
  if (G2 && g2) {
    // the region's next owner clears it before use: this warp's last table
    // stores must be visible device-wide before the release
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicAnd(a.gtab_busy + g2_region / 32, ~(1u << (g2_region % 32)));
  }
}

}  // namespace gann
#include "search_batch.cuh"
namespace gann {

namespace {
template <int E, int M, int LPR, int CPL>
cudaError_t launch_one(const SearchArgs& a0, cudaStream_t s) {
  if (a0.batch_eb) return launch_batch<E, M, LPR, CPL>(a0, s);  // several expansions per step (search_batch.cuh)
  // read per launch (A/B runs flip them between launches)
  const char* dv = std::getenv("GANN_SEARCH_DIAG");
  const bool diag = dv && *dv && *dv != '0';
  const bool f16 = a0.visited_mode == 0 && a0.hash_bits != 0 && !diag;
  // with the second level (G2), no shared table: its 2 KB per warp go to
  // resident warps and the second level answers every neighbour
  // (GANN_GTAB_ONLY=0 keeps both levels)
  const char* go = std::getenv("GANN_GTAB_ONLY");
  SearchArgs a = a0;
  if (f16 && a.gtab && !(go && *go == '0')) a.hash_log2 = 0;
  const uint32_t per_warp = static_cast<uint32_t>(search_smem_per_warp(a.L, a.R, a.hash_log2, a.hash_bits != 0));
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e;
  // CTA width (warps = queries per CTA; the kernel works per warp at any
  // width): the widest whose regions fit the opt-in shared memory, narrowed
  // further while that leaves more warps resident (large beams: 3 CTAs of 4
  // warps at 59 KB each waste 50 KB that 1-warp CTAs use)
  int wpb = kWarpsPerBlock;
  if (const char* wv = std::getenv("GANN_SEARCH_WPB")) wpb = std::max(1, std::min(kWarpsPerBlock, std::atoi(wv)));  // experiment
  while (wpb > 1 && size_t(per_warp) * wpb > static_cast<size_t>(optin)) wpb >>= 1;
  // R = 64 fixed at compile time (measured): 16-lane rows -5% at L=200 (c2)
  // and a faster build search; 8-lane rows (c1): -1% for a serial launch at
  // L=200 but -1% bench QPS (pipelined), +1.4% at L=64, +4.5% for the build's
  // searches — so only the 16-lane instance is specialised
  const char* rv = std::getenv("GANN_SEARCH_R64");
  const bool r64 = a.R == 64 && (rv && *rv ? *rv == '1' : LPR >= 16);
  const bool fit = a.stride == uint64_t(16) * LPR * CPL;
  const bool g2 = a.gtab != nullptr;
  auto k = !f16 ? search_kernel<E, M, LPR, CPL, false>
         : g2 ? (r64 ? (fit ? search_kernel<E, M, LPR, CPL, true, true, true, true>
                            : search_kernel<E, M, LPR, CPL, true, true, false, true>)
                     : (fit ? search_kernel<E, M, LPR, CPL, true, false, true, true>
                            : search_kernel<E, M, LPR, CPL, true, false, false, true>))
              : (r64 ? (fit ? search_kernel<E, M, LPR, CPL, true, true, true> : search_kernel<E, M, LPR, CPL, true, true>)
                     : (fit ? search_kernel<E, M, LPR, CPL, true, false, true>
                            : search_kernel<E, M, LPR, CPL, true, false>));
  if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                size_t(per_warp) * wpb > 48 * 1024 ? static_cast<int>(size_t(per_warp) * wpb)
                                                                   : 48 * 1024)) != cudaSuccess)
    return e;
  if (a.nq == 0) return cudaSuccess;
  if (const char* cv = std::getenv("GANN_SEARCH_CARVE"))  // experiment: shared-memory carve-out, percent
    if ((e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(cv))) != cudaSuccess) return e;
  int per_sm = 0, sms = 0;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, wpb * 32, size_t(per_warp) * wpb)) !=
      cudaSuccess)
    return e;
  if (const char* dv = std::getenv("GANN_BATCH_DEBUG"))
    if (*dv == '1') std::fprintf(stderr, "search launch: L %u per_warp %u wpb %d per_sm %d g2 %d\n", a.L, per_warp, wpb, per_sm, int(g2));
  for (int w = wpb >> 1; w >= 1; w >>= 1) {
    int ps = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, k, w * 32, size_t(per_warp) * w)) != cudaSuccess)
      return e;
    // as many resident warps in narrower CTAs: 2-warp CTAs win the tie (a
    // finishing launch's slots free sooner for the next launch: the bench's
    // pipelined sweep -2 to -3% per launch at L = 10..200, the build unchanged)
    if (ps * w > per_sm * wpb || (w >= 2 && ps * w == per_sm * wpb)) {
      per_sm = ps;
      wpb = w;
    }
  }
  const size_t smem = size_t(per_warp) * wpb;
  const uint32_t want = (a.nq + wpb - 1) / wpb;
  const uint32_t blocks = std::min<uint32_t>(want, static_cast<uint32_t>(std::max(1, per_sm) * sms));
  if ((e = cudaMemsetAsync(a.next_query, 0, sizeof(uint32_t), s)) != cudaSuccess) return e;
  k<<<blocks, wpb * 32, smem, s>>>(a, per_warp);
  return cudaGetLastError();
}

template <int E, int M>
cudaError_t dispatch_geom(const SearchArgs& a, const Geometry& g, cudaStream_t s) {
  switch (g.lpr) {
    case 1: return launch_one<E, M, 1, 1>(a, s);
    case 2: return launch_one<E, M, 2, 1>(a, s);
    case 4: return launch_one<E, M, 4, 1>(a, s);
    case 8: return launch_one<E, M, 8, 1>(a, s);
    case 16: return launch_one<E, M, 16, 1>(a, s);
    default:
      if (g.cpl == 1) return launch_one<E, M, 32, 1>(a, s);
      if (g.cpl == 2) return launch_one<E, M, 32, 2>(a, s);
      return launch_one<E, M, 32, 4>(a, s);
  }
}
}  // namespace

namespace {
template <int E, int M, int LPR, int CPL>
void preload_one() {
  touch_kernel(search_kernel<E, M, LPR, CPL, false>);
  touch_kernel(search_kernel<E, M, LPR, CPL, true, false>);
  touch_kernel(search_kernel<E, M, LPR, CPL, true, true>);
  touch_kernel(search_kernel<E, M, LPR, CPL, true, false, true>);
  touch_kernel(search_kernel<E, M, LPR, CPL, true, true, true>);
  touch_kernel(search_kernel<E, M, LPR, CPL, true, false, false, true>);
  touch_kernel(search_kernel<E, M, LPR, CPL, true, true, false, true>);
  touch_kernel(search_kernel<E, M, LPR, CPL, true, false, true, true>);
  touch_kernel(search_kernel<E, M, LPR, CPL, true, true, true, true>);
  touch_kernel(search_batch_kernel<E, M, LPR, CPL, false>);
  touch_kernel(search_batch_kernel<E, M, LPR, CPL, true>);
}
template <int E, int M>
void preload_geom(const Geometry& g) {
  switch (g.lpr) {
    case 1: return preload_one<E, M, 1, 1>();
    case 2: return preload_one<E, M, 2, 1>();
    case 4: return preload_one<E, M, 4, 1>();
    case 8: return preload_one<E, M, 8, 1>();
    case 16: return preload_one<E, M, 16, 1>();
    default:
      if (g.cpl == 1) return preload_one<E, M, 32, 1>();
      if (g.cpl == 2) return preload_one<E, M, 32, 2>();
      return preload_one<E, M, 32, 4>();
  }
}
}  // namespace

}  // namespace gann
