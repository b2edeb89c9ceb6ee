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
#include "common.cuh"
#include "internal.h"

namespace gann {

// Per-warp shared memory: beam keys (expanded flag in bit 0, merged in place),
// candidate scratch, and the direct-mapped visited table.
size_t search_smem_per_warp(uint32_t L, uint32_t R, uint32_t hash_log2, bool hash16) {
  const size_t Lp = (L + 31) & ~31u, Rp = (R + 31) & ~31u;
  size_t b = Lp * 8 + 2 * Rp * 8 + Rp * 4 + (size_t(1) << hash_log2) * (hash16 ? 2 : 4) + Lp / 8;
  return (b + 15) & ~size_t(15);
}

// Shared memory of the narrowest search CTA: one warp (one query). Wider
// CTAs (up to kSearchWarpsPerBlock) are used while their regions fit.
size_t search_smem_min_block(uint32_t L, uint32_t R, uint32_t hash_log2, bool hash16) {
  return search_smem_per_warp(L, R, hash_log2, hash16);
}

// Per-warp shared memory of search_batch_kernel: beam, candidate keys / ids /
// insertion points / expansion tags for cm candidates per step, merge bitmap.
size_t search_batch_smem_per_warp(uint32_t L, uint32_t cm) {
  const size_t Lp = (L + 31) & ~31u;
  const size_t b = Lp * 8 + size_t(cm) * 8 + size_t(cm) * 4 + 32 + Lp / 8 + size_t(cm) * 2 + size_t(cm) * 2;
  return (b + 15) & ~size_t(15);
}

cudaError_t launch_search_u8(const SearchArgs& a, int metric, const Geometry& g, cudaStream_t s);
cudaError_t launch_search_i8(const SearchArgs& a, int metric, const Geometry& g, cudaStream_t s);
cudaError_t launch_search_f32(const SearchArgs& a, int metric, const Geometry& g, cudaStream_t s);
void preload_search_u8(int metric, const Geometry& g);
void preload_search_i8(int metric, const Geometry& g);
void preload_search_f32(int metric, const Geometry& g);

void preload_search(int elem, int metric, const Geometry& g) {
  if (elem == kU8) return preload_search_u8(metric, g);
  if (elem == kI8) return preload_search_i8(metric, g);
  return preload_search_f32(metric, g);
}

Geometry make_geometry(uint32_t nch) {
  Geometry g{nch, 32, 1};
  if (nch <= 32) {
    int l = 1;
    while (static_cast<uint32_t>(l) < nch) l <<= 1;
    g.lpr = l;
    g.cpl = 1;
  } else {
    g.lpr = 32;
    g.cpl = nch <= 64 ? 2 : 4;
  }
  return g;
}

cudaError_t launch_search(const SearchArgs& a, int elem, int metric, const Geometry& g,
                          cudaStream_t s) {
  if (elem == kU8) return launch_search_u8(a, metric, g, s);
  if (elem == kI8) return launch_search_i8(a, metric, g, s);
  return launch_search_f32(a, metric, g, s);
}

}  // namespace gann
