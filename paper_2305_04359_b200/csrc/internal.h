// internal.h — argument blocks and launchers shared between the kernel
// translation units and the C-ABI host code (gann.cu). Not installed.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace gann {

void set_last_error(const std::string& msg);  // gann_last_error() text (gann.cu)
// checked builds (common.cuh GANN_CHECK): each kernel translation unit's
// largest failing check line (0: none, or a release build)
unsigned check_line_search_u8();
unsigned check_line_search_i8();
unsigned check_line_search_f32();
unsigned check_line_prune();
unsigned check_line_backedge();
unsigned check_line_misc();

// Row geometry: LPR lanes per row, up to CPL 16-byte chunks per lane.
struct Geometry {
  uint32_t nch;  // 16-byte chunks per (padded) row
  int lpr;       // 1, 2, 4, 8, 16 or 32
  int cpl;       // 1..4 (only with lpr == 32)
};
Geometry make_geometry(uint32_t nch);

// The graph as the kernels see it. Unpartitioned: one table, adj holds every
// row. Vertex-partitioned (one partition per GPU): rows [base, base + P) live
// in this GPU's adj; any row can be read through parts[v / P] (peer / IPC
// pointers), writes go to owned rows only.
struct GraphView {
  uint32_t* adj;                 // local rows
  const uint32_t* const* parts;  // nparts row-storage pointers (device table)
  uint32_t part_size;            // P
  uint32_t nparts;
  uint32_t base;                 // first locally owned vertex
};
__device__ __forceinline__ const uint32_t* graph_row(const GraphView& g, uint32_t v, uint32_t R) {
  if (g.nparts == 1) return g.adj + static_cast<uint64_t>(v) * R;
  return g.parts[v / g.part_size] + static_cast<uint64_t>(v % g.part_size) * R;
}
__device__ __forceinline__ uint32_t* local_row(const GraphView& g, uint32_t v, uint32_t R) {
  return g.adj + static_cast<uint64_t>(v - g.base) * R;
}

enum StatIdx {
  kStQueries = 0, kStExpansions, kStEvals, kStDrops, kStAdj,
  kStPruneLists, kStPruneCands, kStPruneEvals, kStMerges, kStSurvivors, kStMoved, kStDups, kStGuess, kStCount
};

// The counters are replicated kStatSlots times (a prune CTA adds to slot
// blockIdx % kStatSlots; gann_get_stats sums the slots): one set of addresses
// took every list's atomics, and at ~130M lists per c1 build their
// serialisation at L2 cost the re-prune phase 15% (797 -> 679 ms). The search
// kernels (three adds per query) stay on slot 0: the slot arithmetic cost
// search_kernel its 72nd-register budget (73 registers: 6 CTAs instead of 7,
// build search phase 1447 -> 1594 ms).
constexpr uint32_t kStatSlots = 64;
#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long* stat_slot(unsigned long long* stats) {
  return stats + (blockIdx.x % kStatSlots) * kStCount;
}
#endif

struct SearchArgs {
  const uint8_t* data;       // n rows of `stride` bytes
  uint64_t stride;
  uint32_t n;
  GraphView graph;           // n rows of R ids, kNone padded
  uint32_t R;
  uint32_t start;
  const uint8_t* queries;    // nq rows of `stride` bytes (when query_rows == nullptr)
  const uint32_t* query_rows;// build mode: query i is data row query_rows[i]
  const uint32_t* start_override;
  uint32_t nq;
  uint32_t L, k_gate, k_out;
  float eps;
  int visited_mode;          // 0 fast (shared table), 1 reference L*L table, 2 exact set
  uint32_t exact_slots;      // mode 2: slots per query (power of two)
  uint32_t hash_log2;        // fast mode table size (entries)
  uint32_t hash_bits;        // fast mode: 0 = u32 id slots; else u16 remainders of a
                             // bijective hash over hash_bits bits: direct mapped
                             // (hash_ways 1: hash_log2 + 15 bits) or 2-way buckets of
                             // two u16 slots (hash_ways 2: hash_log2 + 14 bits)
  uint32_t hash_ways;
  uint32_t* ref_table;       // modes 1/2: per-query tables, initialised by the kernel
  uint32_t dim;              // real dimension (search_seed)
  uint32_t row_bytes;        // real bytes per row (search_seed)
  uint32_t* out_ids;         // nq * k_out (nullable)
  float* out_dists;
  uint32_t* n_visited;       // nq (nullable)
  uint64_t* dist_comps;      // nq (nullable)
  uint32_t* vis_ids;         // nq * vcap (nullable)
  float* vis_dists;
  uint32_t vcap;
  uint32_t* overflow;        // count of searches whose |V| exceeded vcap
  uint32_t* next_query;      // persistent warps: dynamic query counter (zeroed per launch)
  unsigned long long* stats; // kStCount counters (nullable)
  // second-level visited tables (fast mode, large beams; nullable): regions of
  // 2^gtab_log2 u64 buckets (4 u16 remainders each) in global memory, mostly
  // L2-resident; a warp claims a free region through the gtab_busy bitmap
  // (gtab_regions bits) and searches without one if none is free
  uint64_t* gtab;
  uint32_t* gtab_busy;
  uint32_t gtab_regions;
  uint32_t gtab_log2;
  int gtab_keep;             // second-level table accesses carry an L2 evict_last policy
  int gtab_wide;             // search_batch_kernel: buckets of two u32 ids (n beyond the remainders' reach)
  int next_pf;               // prefetch the next expansion's row before the merge
  // several expansions per step (search_batch.cuh; Alg. 1 form, fast mode, R <= 64):
  uint32_t batch_eb;         // expansions tried per step (0: one per step, search_kernel)
  uint32_t batch_cm;         // fresh ids a step holds (multiple of 32, <= 256)
  int batch_policy;          // 0: always batch_eb; 1: committed + 1; 2: batch_eb after a full commit, else committed + 1
};
constexpr uint32_t kGtabLog2 = 12;  // largest region: 4096 buckets x 4 slots = 16k ids, 32 KB
constexpr uint32_t kGtabLog2Default = 11;  // 8k ids, 16 KB: c1 L=832 evaluations 9.5k -> 11.9k per query, DRAM 36 -> 23 GB per launch, -2%
size_t search_smem_per_warp(uint32_t L, uint32_t R, uint32_t hash_log2, bool hash16);
constexpr int kSearchWarpsPerBlock = 4;  // one query per warp
size_t search_smem_min_block(uint32_t L, uint32_t R, uint32_t hash_log2, bool hash16);
size_t search_batch_smem_per_warp(uint32_t L, uint32_t cm);  // search_batch_kernel (search_batch.cuh)

// Kernel preloading. CUDA loads a kernel's code at its first launch (lazy
// module loading), which put 15-200 ms of one-time stalls into the first
// build of a process; index creation touches the kernels the index will use
// (cudaFuncGetAttributes) so the build and the searches start warm.
void preload_search(int elem, int metric, const Geometry& g);
void preload_prune(int elem, int metric, const Geometry& g);
void preload_backedge(int elem, int metric, const Geometry& g);
void preload_misc(int elem, int metric);
template <class K>
inline void touch_kernel(K k) {
  cudaFuncAttributes attr;
  (void)cudaFuncGetAttributes(&attr, reinterpret_cast<const void*>(k));
}
cudaError_t launch_search(const SearchArgs& a, int elem, int metric, const Geometry& g,
                          cudaStream_t s);

// The tensor-core prune's stage-1 -> stage-2 hand-off region. One per index
// (host-side bookkeeping; kernels only see the device pointer), so two
// indexes pruning on one device from different host threads never share it.
struct PruneHandoff {
  uint32_t* buf = nullptr;
  uint64_t cap = 0;
};

struct PruneArgs {
  const uint8_t* data;
  uint64_t stride;
  uint32_t count;              // lists
  const uint32_t* list_index;  // nullable: list i of this launch is list_index[i]
  const uint32_t* points;      // p per list
  const uint64_t* begins;      // list l starts at begins[l] (nullable => l*fixed_stride)
  uint64_t fixed_stride;
  const uint32_t* lengths;     // list l has lengths[l] candidates
  const uint32_t* cand_ids;
  const float* cand_dists;
  uint32_t R;
  float alpha;
  int rule;                    // 0 scale_candidate, 1 scale_selected
  uint32_t* out_adj;           // write to out_adj[(p - out_base) * R] (when out_rows == nullptr)
  uint32_t out_base;
  uint32_t* out_rows;          // or to out_rows[l * R]
  uint32_t* n_out;             // nullable, per list l
  uint32_t mcap;               // max list length this launch supports
  uint32_t mmin;               // lists shorter than this are left to another launch
  int skip_long;               // lists longer than mcap: skip silently (binned launches)
  uint32_t* too_long;          // ... or count them here
  unsigned long long* stats;
  // Per graph row: how many leading entries are a prune's output (<= 255;
  // mutually non-culling). Written by every kernel that writes a row into
  // out_adj (nullable). With row_lists set, a list of this launch starts with
  // its point's current row, so that prefix needs no pair tests among itself.
  uint8_t* spre;
  int row_lists;
  PruneHandoff* hand;          // host pointer: the calling index's hand-off region
  // bin_lists: re-prune lists (row_lists) whose row prefix leaves at most
  // small_u other entries go to an extra bin (index nb) for the warp kernel
  uint32_t small_u;
  uint32_t small_u2;           // ... and those with at most small_u2 of them to bin nb, the rest of the class to nb + 1
};
// threads = 32 for short lists, larger for hubs; smem from prune_smem_bytes.
size_t prune_smem_bytes(uint32_t mcap, uint32_t R);
cudaError_t launch_prune(const PruneArgs& a, int elem, int metric, const Geometry& g, int threads,
                         cudaStream_t s);
// Length bins: lists[b * count + i] for i < counts[b], b over bounds (last bin: longer).
cudaError_t launch_bin_lists(const PruneArgs& a, const uint32_t* d_bounds, int nb, uint32_t* d_counts,
                             uint32_t* d_lists, cudaStream_t s);
// Re-prunes of a row prefix plus <= small_u entries (integer rows, R <= 64):
// one warp per list (prune.cu reprune_small_kernel).
uint32_t reprune_small_max_u();
uint32_t reprune_small_low_u();
cudaError_t launch_reprune_small(const PruneArgs& a, int elem, int metric, const Geometry& g, cudaStream_t s);
// Integer lists up to 512 candidates run on the tensor cores (IMMA tiles).
bool prune_uses_mma(int elem, uint32_t mcap, uint64_t stride, uint32_t R);
// Allocate the tensor-core prune's hand-off region up front for launches of
// up to `lists` lists (a build sizes it once from its largest batch).
void prune_reserve(PruneHandoff* h, uint32_t lists, uint64_t stride, uint32_t R, cudaStream_t s);
void prune_release(PruneHandoff* h, cudaStream_t s);  // frees an index's hand-off region

// ---- back-edge grouping (phase 2) -----------------------------------------
// Pairs (target, source) come either from the out-rows of the batch's points
// (batch form: pair e = (adj[bsrc[e/R]*R + e%R], bsrc[e/R]), the reference's
// concatenation order, src/diskann.cpp:61-65) or from explicit arrays.
struct BackEdgeArgs {
  const uint8_t* data;
  uint64_t stride;
  uint32_t* adj;            // locally owned rows (vertex v at (v - base) * R)
  uint32_t base;            // first owned vertex; tcount/tgroup are indexed by v - base
  uint32_t R;
  const uint32_t* bsrc;     // batch form: B source points
  uint32_t B;
  const uint32_t* ptarget;  // explicit form (nullable): targets
  const uint32_t* psource;  //                           sources
  const uint32_t* pordinal; // explicit form: order key of each pair (nullable = its index)
  uint32_t pstride;         // element stride of ptarget / pordinal (interleaved pairs: 2)
  uint64_t npairs;          // B*R (batch form) or explicit count
  int sources_distinct;     // batch form: every source appears once per target
  uint32_t* tcount;         // n, all zero on entry and on exit
  uint32_t* tgroup;         // n
  uint32_t* gtarget;        // per group
  uint32_t* gcnt;
  uint64_t* goff;           // ordinal slots of group g: [goff[g], goff[g]+gcnt[g])
  uint32_t* gcursor;
  uint32_t* gsrc;           // npairs ordinals
  uint64_t* poff;           // merged-list region of group g (R + gcnt[g] slots)
  uint32_t* plen;           // merged length
  uint32_t* pid;            // merged ids
  float* pdist;             // d(target, id)
  unsigned long long* counters;  // see kCnt*
  uint32_t* big_groups;     // groups with more than small_group_cap sources
  uint32_t* plist_small;    // groups to re-prune, merged length <= prune_small_cap
  uint32_t* plist_big;
  const uint32_t* key_of_target; // group_by_key: real key of a dense target slot
  uint32_t small_group_cap;
  uint32_t big_group_cap;
  uint32_t prune_small_cap;
  int small_dists;          // stage d(t, .) for small lists too (else the prune computes them)
};
enum { kCntGroups = 0, kCntPairsCursor, kCntPruneCursor, kCntBig, kCntMaxGroup,
       kCntPruneSmall, kCntPruneBig, kCntMaxMerged, kCntTooBig, kCntNum };
cudaError_t backedge_count(const BackEdgeArgs& a, cudaStream_t s);
cudaError_t backedge_offsets(const BackEdgeArgs& a, uint32_t ngroups, cudaStream_t s);
cudaError_t backedge_scatter(const BackEdgeArgs& a, cudaStream_t s);
cudaError_t backedge_merge(const BackEdgeArgs& a, uint32_t ngroups, uint32_t nbig, int elem,
                           int metric, const Geometry& g, cudaStream_t s);
size_t backedge_merge_smem(uint32_t cap, uint32_t R);
// group_by_key: map arbitrary u32 keys to dense slots of a 2^k-entry table.
cudaError_t launch_hash_keys(const uint32_t* keys, uint64_t m, uint32_t* table, uint32_t tbits,
                             uint32_t* slots, cudaStream_t s);
// group_by_key output: pairs of group g written at [goff[g], goff[g]+gcnt[g]).
cudaError_t backedge_write_groups(const BackEdgeArgs& a, uint32_t ngroups, uint32_t nbig,
                                  uint32_t* out_keys, uint32_t* out_vals, cudaStream_t s);

// ---- vertex-partitioned build: reverse pairs routed to the target's owner ------
// Pair k of local inserted point (ids[k], batch offset bo[k]) and out-slot i:
// (target, bo*R + i) sent to partition target / P. counts/offsets: nparts u64.
cudaError_t part_pairs_count(const uint32_t* adj_local, uint32_t base, uint32_t R, const uint32_t* ids,
                             uint32_t K, uint32_t P, unsigned long long* counts, cudaStream_t s);
cudaError_t part_pairs_scatter(const uint32_t* adj_local, uint32_t base, uint32_t R, const uint32_t* ids,
                               const uint32_t* bo, uint32_t K, uint32_t P, unsigned long long* cursors,
                               uint32_t* out_pairs, cudaStream_t s);

// ---- misc -------------------------------------------------------------------
cudaError_t launch_choose_start(const uint8_t* data, uint64_t stride, uint64_t n, uint32_t d,
                                int elem, int metric, double* colsum, float* centroid,
                                unsigned long long* best, cudaStream_t s);
// table[u] = Phi^-1((u + 1/2) / 2^16) on a 2^-16 grid (host, 65536 floats)
void normal_table(float* out);
const float* device_normal_table();
cudaError_t launch_generate_f32(float* out, uint64_t n, uint32_t d, uint32_t clusters, float sigma,
                                float norm_sigma, float shift, uint64_t center_seed, uint64_t stream_seed,
                                uint64_t row0, cudaStream_t s);
cudaError_t launch_generate_u8(uint8_t* out, uint64_t out_stride, uint64_t n, uint32_t d,
                               uint32_t clusters, float sigma, float noise_frac,
                               uint64_t center_seed, uint64_t stream_seed, uint64_t row0,
                               cudaStream_t s);
cudaError_t launch_groundtruth(const uint8_t* data, uint64_t stride, uint64_t n,
                               const uint8_t* queries, uint32_t nq, uint32_t k, int elem,
                               int metric, uint32_t nch, unsigned long long* partial,
                               uint32_t splits, uint32_t* ids, float* dists, cudaStream_t s);
uint32_t groundtruth_splits(uint64_t n, uint32_t nq);
cudaError_t stable_sort_pairs_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                                  uint32_t* vals_out, uint64_t m, int bits, void** tmp, size_t* tmp_bytes,
                                  cudaStream_t s);
// The shuffled insertion order from std::shuffle's swap log r (misc.cu): out[0..n), front in slot 0;
// work: 4 n u32 of device scratch.
cudaError_t launch_shuffle_from_log(const uint32_t* r, uint64_t n, uint32_t front, uint32_t* work, uint32_t* out,
                                    void** tmp, size_t* tmp_bytes, cudaStream_t s);
// Validate rows [0, rows) of an n-vertex graph (row r is vertex row0 + r):
// *bad = ~0 if fine, else (first bad row << 3) | code (1 id after padding,
// 2 id out of range, 3 self loop, 4 repeated id).
cudaError_t launch_validate_rows(const uint32_t* adj, uint64_t rows, uint32_t R, uint64_t n, uint64_t row0,
                                 unsigned long long* bad, cudaStream_t s);

}  // namespace gann
