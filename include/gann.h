/* gann.h — C ABI of the B200-native Vamana batch build + batched beam search.
 *
 * This is the drop-in boundary for the hot path of the reference (graphann,
 * arXiv 2305.04359). Every entry point takes plain pointers and sizes; no
 * torch or CUDA types cross it. Each function cites the reference interface it
 * replaces (paths relative to the reference's proj/ directory).
 *
 * Conventions
 *   elem     GANN_U8 / GANN_I8 / GANN_F32         (graphann::ElemKind, include/graphann/core.hpp:23)
 *   metric   GANN_L2 (squared) / GANN_IP (negated) (graphann::Metric, include/graphann/metric.hpp:13)
 *   rule     GANN_SCALE_CANDIDATE / GANN_SCALE_SELECTED (graphann::PruneRule, include/graphann/prune.hpp:19)
 *   graph    n rows of R uint32 ids; unused slots hold GANN_NONE and the
 *            degree of a row is the length of its non-GANN_NONE prefix
 *            (graphann::NeighborGraph, include/graphann/graph.hpp:16-59).
 *   results  ids padded with GANN_NONE, distances with +inf.
 *   errors   return GANN_OK (0); GANN_EINVAL (1) where the reference throws
 *            std::invalid_argument; GANN_EIO (2) for io_error/format_error;
 *            GANN_ECUDA (3) for a CUDA failure. gann_last_error() returns the
 *            calling thread's message.
 *   threads  calls on one gann_index are serialised by the caller (the index
 *            owns one CUDA stream); different indexes may be used from
 *            different host threads.
 *   host vs device: functions without a _device suffix take HOST buffers and
 *            are synchronous, like the reference's by-value returns. The
 *            _device variants take device pointers and enqueue on `stream`
 *            (NULL = the index's stream) without synchronising.
 */
#ifndef GANN_H
#define GANN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GANN_NONE 0xFFFFFFFFu

enum { GANN_U8 = 0, GANN_I8 = 1, GANN_F32 = 2 };
enum { GANN_L2 = 0, GANN_IP = 1 };
enum { GANN_SCALE_CANDIDATE = 0, GANN_SCALE_SELECTED = 1 };
/* Visited filter of the search kernel. FAST: a bounded shared-memory hash
 * with no false positives (ids, visit order and |V| are identical to the
 * reference; dist_comps counts this kernel's own evaluations). REF: the
 * reference's L*L-slot ApproxVisitedSet (include/graphann/search.hpp:24-38)
 * held in global memory, so dist_comps matches the reference too. */
/* EXACT: an exact seen-set per query in global memory (never forgets), so
 * dist_comps counts distinct evaluated ids — the U of SURVEY.md §8d. */
enum { GANN_VISITED_FAST = 0, GANN_VISITED_REF = 1, GANN_VISITED_EXACT = 2 };
enum { GANN_OK = 0, GANN_EINVAL = 1, GANN_EIO = 2, GANN_ECUDA = 3 };

typedef struct gann_index gann_index;

const char* gann_last_error(void);
/* Library/ABI version string, e.g. "gann 0.1 sm_100a". */
const char* gann_version(void);

/* ---- index lifetime -------------------------------------------------------
 * Replaces graphann::VectorDataset (include/graphann/dataset.hpp:16) +
 * NeighborGraph(n, cap) (include/graphann/graph.hpp:20): uploads the points
 * into an HBM-resident, 16-byte-padded row layout and allocates an empty graph
 * of capacity R. */
int gann_index_create(const void* points, uint64_t n, uint32_t d, int elem, int metric,
                      uint32_t R, int device, gann_index** out);
/* Same, from points already resident on `device` (row-major, d*elem bytes). */
int gann_index_create_device(const void* d_points, uint64_t n, uint32_t d, int elem,
                             int metric, uint32_t R, int device, gann_index** out);
void gann_index_free(gann_index* idx);
int gann_index_info(const gann_index* idx, uint64_t* n, uint32_t* d, int* elem, int* metric,
                    uint32_t* R, uint32_t* start);

/* ---- build ----------------------------------------------------------------
 * Replaces graphann::build_diskann(ds, metric, DiskannParams{R, L, alpha, rule,
 * seed}, workers) (include/graphann/diskann.hpp:36-37, src/diskann.cpp:31-70).
 * max_batch = 0 reproduces the reference's uncapped prefix-doubling schedule
 * (src/builder_common.cpp:13-20); max_batch > 0 caps every batch at
 * hi = min(2*lo, lo + max_batch, n). */
int gann_build(gann_index* idx, uint32_t L, float alpha, int rule, uint64_t seed,
               uint32_t max_batch);
/* create + build in one call: the reference's build(points, R, L, alpha). */
int gann_build_diskann(const void* points, uint64_t n, uint32_t d, int elem, int metric,
                       uint32_t R, uint32_t L, float alpha, int rule, uint64_t seed,
                       uint32_t max_batch, int device, gann_index** out);

/* Graph transfer (NeighborGraph::out_neighbors/set_neighbors/start,
 * include/graphann/graph.hpp:29-45; the ANNG payload of src/graph.cpp:96-178).
 * import validates ids (< n, no self loops) like set_neighbors
 * (src/graph.cpp:42-59). deg may be NULL on export. */
int gann_import_graph(gann_index* idx, const uint32_t* adj, uint32_t start);
/* Device-resident rows (n*R, GANN_NONE padded), copied as is (trusted: no
 * validation) — e.g. the rows all-gathered from a partitioned build. */
int gann_import_graph_device(gann_index* idx, const uint32_t* d_adj, uint32_t start);
int gann_export_graph(const gann_index* idx, uint32_t* adj, uint32_t* deg, uint32_t* start);

/* ---- search ---------------------------------------------------------------
 * Replaces graphann::beam_search(g, ds, metric, q, SearchParams{L, k_gate, eps},
 * counter, start_override) (include/graphann/search.hpp:57-60,
 * src/search.cpp:62-131) for a batch of nq queries. k_gate is the
 * reference's SearchParams::k (expansion gate); k_gate = L is the plain
 * Alg. 1 drain used by insert_point. Outputs the k_out best of the visited
 * set (k_out <= L), |V| and dist_comps per query (both nullable), and
 * optionally the visited sequence (vis_ids/vis_dists, vcap per query,
 * nullable). start_override (nullable) gives one start per query. */
int gann_search(gann_index* idx, const void* queries, uint32_t nq, uint32_t k_out, uint32_t L,
                uint32_t k_gate, float eps, int visited_mode, const uint32_t* start_override,
                uint32_t* ids, float* dists, uint32_t* n_visited, uint64_t* dist_comps,
                uint32_t* vis_ids, float* vis_dists, uint32_t vcap);
/* Device-pointer variant (queries row-major d*elem bytes on the device). */
int gann_search_device(gann_index* idx, const void* d_queries, uint32_t nq, uint32_t k_out,
                       uint32_t L, uint32_t k_gate, float eps, int visited_mode,
                       uint32_t* d_ids, float* d_dists, uint32_t* d_n_visited,
                       uint64_t* d_dist_comps, void* stream);
/* The largest beam L this index's search kernel holds on chip (beam, candidate
 * lists and visited table of a query live in shared memory; L above it is
 * rejected with GANN_EINVAL). The reference has no such limit. */
int gann_search_max_beam(const gann_index* idx, uint32_t* max_L);
/* Stage a query batch once (padded device layout) so repeated
 * gann_search_staged calls time only the search kernel. */
int gann_stage_queries(gann_index* idx, const void* d_queries, uint32_t nq);
int gann_search_staged(gann_index* idx, uint32_t k_out, uint32_t L, uint32_t k_gate, float eps,
                       uint32_t* d_ids, float* d_dists, void* stream);
/* Serving form of gann_search (fast visited mode): everything is enqueued on
 * `stream` and the call returns at once; results are in h_ids / h_dists
 * (nq*k_out, pinned host memory for a truly asynchronous copy) when the
 * stream has reached this point. All per-call device state lives in the
 * caller's d_scratch (gann_search_async_scratch bytes), so calls on different
 * streams may run concurrently: a batch's tail overlaps the next batch. The
 * index itself is only read (synchronise those streams before
 * gann_index_free). */
uint64_t gann_search_async_scratch(const gann_index* idx, uint32_t nq, uint32_t k_out);
int gann_search_async(gann_index* idx, const void* h_queries, uint32_t nq, uint32_t k_out,
                      uint32_t L, uint32_t k_gate, float eps, uint32_t* h_ids, float* h_dists,
                      void* d_scratch, uint64_t scratch_bytes, void* stream);

/* ---- the build's internals, individually (parity + reuse) ------------------
 * alpha_prune: graphann::alpha_prune (include/graphann/prune.hpp:31-33,
 * src/prune.cpp:8-44) over `count` candidate lists at once. List i has point
 * p[i] and candidates cand_ids/cand_dists[offsets[i] .. offsets[i+1]). The
 * kept ids of list i go to out[i*R ..] (GANN_NONE padded); n_out[i] = count. */
int gann_alpha_prune(gann_index* idx, const uint32_t* p, const uint64_t* offsets,
                     uint32_t count, const uint32_t* cand_ids, const float* cand_dists,
                     float alpha, int rule, uint32_t* out, uint32_t* n_out);
/* group_by_key: graphann::group_by_key (include/graphann/semisort.hpp:21-22,
 * src/semisort.cpp:15-73) on the GPU. Equal keys are contiguous, input order is
 * kept inside a group; group order is unspecified (as in the reference, where it
 * is hash-bucket order). offsets has n_groups+1 entries. */
int gann_group_by_key(const uint32_t* keys, const uint32_t* vals, uint64_t m, int device,
                      uint32_t* out_keys, uint32_t* out_vals, uint64_t* offsets,
                      uint64_t* n_groups);
/* choose_start: graphann::choose_start (src/builder_common.cpp:58-97). */
int gann_choose_start(gann_index* idx, uint32_t* start);
/* insert_point over a batch: graphann::insert_point (src/diskann.cpp:12-29) for
 * points ids[0..count) against the current graph (all read the same
 * snapshot, as in one build batch). Writes each out-list into the graph and,
 * if back != NULL, copies it to back[i*R ..] (the reverse-edge targets). */
int gann_insert_batch(gann_index* idx, const uint32_t* ids, uint32_t count, uint32_t L,
                      float alpha, int rule, uint32_t* back);
/* apply_back_edges: graphann::apply_back_edges (src/builder_common.cpp:109-140). */
int gann_apply_back_edges(gann_index* idx, const uint32_t* targets, const uint32_t* sources,
                          uint64_t m, float alpha, int rule);

/* Host helpers of the build schedule (no device work):
 * shuffled_order — graphann::shuffled_order (src/builder_common.cpp:99-107),
 *   the same libstdc++ std::mt19937_64 + std::shuffle draw;
 * batch_ranges — graphann::batch_ranges (src/builder_common.cpp:13-20) with the
 *   optional cap; returns the number of ranges (writes at most max_ranges). */
void gann_shuffled_order(uint32_t n, uint64_t seed, uint32_t front, uint32_t* out);
/* std::shuffle's swap log for (n, seed): log[i] is the position the same
 * libstdc++ call swaps element i with (log[0] = 0), i.e. shuffled_order before
 * its front swap is `a = iota; for i in 1..n-1: swap(a[i], a[log[i]])`. gann_build
 * draws this log on the host and resolves the permutation on the device. */
void gann_shuffle_swap_log(uint32_t n, uint64_t seed, uint32_t* log);
uint32_t gann_batch_ranges(uint64_t n, uint32_t max_batch, uint32_t* lo, uint32_t* hi,
                           uint32_t max_ranges);
/* The seed build_diskann derives for shuffled_order: mix64(seed, "insert"). */
uint64_t gann_insert_seed(uint64_t seed);

/* ---- files in the reference's formats ----------------
 * Graph: graphann's ANNG layout (src/graph.cpp:96-178): "ANNG", u32 version 1,
 * u32 n, u32 capacity, u32 start, u32 degrees[n], then the live ids in vertex
 * order. load validates like graphann::load_graph (magic, version, start,
 * degree <= capacity, ids, self loops, duplicates, trailing bytes) and returns
 * GANN_EIO on a malformed file; the file's capacity must not exceed R.
 * Vectors: graphann::load_vectors (src/dataset.cpp:71-122): .u8bin/.i8bin/.fbin
 * ("bin": u32 n, u32 d, payload) and .bvecs/.fvecs ("vecs": per-vector u32 d
 * prefix); the element kind comes from the extension. */
int gann_save_graph(const gann_index* idx, const char* path);
int gann_load_graph(gann_index* idx, const char* path);
int gann_index_create_from_file(const char* path, int metric, uint32_t R, int device,
                                gann_index** out);

/* ---- range search --------------------------------------
 * graphann::range_search (src/search.cpp:133-149): the drained beam {L, L, eps}
 * then every visited vertex with dist <= r^2 (L2) or <= r (IP), ascending
 * (dist, id). Query q's results go to ids/dists[q*cap ..]; counts[q] is the
 * full count (it may exceed cap). */
int gann_range_search(gann_index* idx, const void* queries, uint32_t nq, float radius, uint32_t L,
                      float eps, uint32_t cap, uint32_t* counts, uint32_t* ids, float* dists);

/* ---- layered (HNSW) search ------------------------------
 * graphann::search_hnsw (src/hnsw.cpp:130-147) over a layered index: layer 0 is
 * `layer0` (its points and bottom graph, borrowed: it must outlive the handle);
 * layers 1..num_layers-1 are graphs over the same id space, rows of
 * `m_upper` ids (GANN_NONE padded; non-members have empty rows), layer l at
 * upper_adj[((l-1)*n + v)*m_upper]. `entry` is the top layer's entry vertex
 * (HnswIndex::entry, include/graphann/hnsw.hpp). A query descends with beam
 * {1, 1, 0} searches from `entry`, each layer started at the previous layer's
 * nearest, then searches layer 0 with {L, k_gate, eps} from there.
 * dist_comps sums every layer's evaluations, as the reference does. */
typedef struct gann_hnsw gann_hnsw;
int gann_hnsw_create(gann_index* layer0, uint32_t num_layers, const uint32_t* upper_adj, uint32_t m_upper,
                     uint32_t entry, gann_hnsw** out);
int gann_hnsw_search(gann_hnsw* h, const void* queries, uint32_t nq, uint32_t k_out, uint32_t L,
                     uint32_t k_gate, float eps, int visited_mode, uint32_t* ids, float* dists,
                     uint32_t* n_visited, uint64_t* dist_comps);
void gann_hnsw_free(gann_hnsw* h);

/* ---- next-row helpers --------------------------------------
 * Exact top-k by (dist, id): graphann::compute_groundtruth (src/dataset.cpp:172-217).
 * k <= 64, rows up to 1568 bytes (integer kinds: distances identical to the
 * reference's; f32: FMA partial sums, within the search's f32 tolerance). */
int gann_groundtruth(gann_index* idx, const void* queries, uint32_t nq, uint32_t k,
                     uint32_t* ids, float* dists);
int gann_groundtruth_device(gann_index* idx, const void* d_queries, uint32_t nq, uint32_t k,
                            uint32_t* d_ids, float* d_dists, void* stream);

/* Seeded synthetic u8 Gaussian-mixture rows (BASELINE configs 0-2, 4) written
 * straight into device memory: rows [row0, row0+n) of the stream `stream_seed`,
 * cluster centres from `center_seed`. Pure function of its arguments. */
int gann_generate_u8(void* d_out, uint64_t n, uint32_t d, uint32_t clusters, float sigma,
                     float noise_frac, uint64_t center_seed, uint64_t stream_seed, uint64_t row0,
                     int device);
/* The generators' normal deviates: out[u] = Phi^-1((u + 1/2) / 2^16) for
 * u < 65536, on a 2^-16 grid (host only, no GPU needed). A deviate is
 * out[hash & 0xFFFF]: an exact Gaussian up to the 16-bit discretisation. */
int gann_normal_table(float* out);
/* Seeded synthetic f32 rows (BASELINE config 3, TTI-like): a `clusters`-
 * component mixture, v = c + sigma z (c, z ~ N(0, 1), gann_normal_table), scaled
 * to norm exp(norm_sigma g) (log-normal per-point norms); shift > 0 moves
 * every centre by shift * N(0, 1) (the out-of-distribution query set).
 * Computed in double, rounded to f32 once. */
int gann_generate_f32(void* d_out, uint64_t n, uint32_t d, uint32_t clusters, float sigma,
                      float norm_sigma, float shift, uint64_t center_seed, uint64_t stream_seed,
                      uint64_t row0, int device);

/* ---- vertex-partitioned build (BASELINE config 4) -----------
 * One index per GPU (one process per GPU). Every index holds all points;
 * partition `rank` of `nparts` owns graph rows [rank*P, min(n, (rank+1)*P)),
 * P = ceil(n / nparts). Peers' rows are read through CUDA IPC mappings
 * (NVLink peer memory on a multi-GPU node). Per build batch the caller runs
 *   phase1   -> insert this partition's points of the batch; returns the
 *               reverse pairs (target, batch ordinal) grouped by owner
 *               (interleaved u32 pairs in device memory, counts[nparts]);
 *   exchange -> all-to-all-v of the pairs (NCCL), receive concatenated;
 *   phase2   -> merge the received pairs into the owned rows;
 *   barrier  -> before the next batch's searches.
 * The result equals the single-GPU build row for row. export_graph returns a
 * partition's own rows. */
int gann_index_create_part(const void* points, uint64_t n, uint32_t d, int elem, int metric,
                           uint32_t R, uint32_t rank, uint32_t nparts, int device, gann_index** out);
/* d_points may be NULL: the index's points are then zero for the caller to
 * fill in place (gann_index_device_ptrs), so 1B points need no second copy. */
int gann_index_create_part_device(const void* d_points, uint64_t n, uint32_t d, int elem, int metric,
                                  uint32_t R, uint32_t rank, uint32_t nparts, int device,
                                  gann_index** out);
int gann_part_info(const gann_index* idx, uint32_t* rank, uint32_t* nparts, uint64_t* base,
                   uint64_t* rows);
int gann_part_ipc_handle(const gann_index* idx, void* handle64);
int gann_part_attach(gann_index* idx, uint32_t rank, const void* handle64);
int gann_part_build_begin(gann_index* idx, uint32_t L, float alpha, int rule, uint64_t seed,
                          uint32_t max_batch, uint32_t* nbatches);
int gann_part_phase1(gann_index* idx, uint32_t batch, uint64_t* counts, const uint32_t** d_pairs);
int gann_part_phase2(gann_index* idx, uint32_t batch, const uint32_t* d_pairs, uint64_t m);

/* The collectives of a partitioned build, supplied by the caller (one per
 * rank). Every callback returns 0 on success. `stream` is the index's CUDA
 * stream (cudaStream_t); device buffers hold interleaved u32 pairs (8 bytes a
 * pair), counts are in pairs.
 *   alltoall_counts: send[nranks] -> recv[nranks] (host arrays)
 *   alltoallv:       d_send holds send_counts[g] pairs for rank g, in rank
 *                    order; d_recv receives recv_counts[g] pairs from rank g,
 *                    in rank order (device pointers)
 *   barrier:         all ranks' work queued so far is complete
 * gann_exchange_nccl fills one from an NCCL communicator; any transport with
 * these semantics works (the tests drive it with torch.distributed/gloo). */
typedef struct gann_exchange {
  void* ctx;
  uint32_t rank, nranks;
  int (*alltoall_counts)(void* ctx, const uint64_t* send, uint64_t* recv);
  int (*alltoallv)(void* ctx, const void* d_send, const uint64_t* send_counts, void* d_recv,
                   const uint64_t* recv_counts, void* stream);
  int (*barrier)(void* ctx, void* stream);
} gann_exchange;

/* The whole vertex-partitioned build of build_diskann (src/diskann.cpp:31-70):
 * begin + per batch phase1 -> exchange -> phase2 -> barrier, driven in C++.
 * Collective: every rank calls it with the same parameters. */
int gann_part_build(gann_index* idx, const gann_exchange* x, uint32_t L, float alpha, int rule, uint64_t seed,
                    uint32_t max_batch, uint64_t* pairs_sent);
/* The largest global batch (points, all ranks together) whose build scratch
 * fits `budget_bytes` on each rank, for build beam L; a cap for max_batch at
 * 1B points (0.2-0.5% of n instead of 2%). */
int gann_part_batch_cap(const gann_index* idx, uint32_t L, uint64_t budget_bytes, uint32_t* max_batch);

/* NCCL (loaded at run time: the libnccl.so.2 already in the process, e.g.
 * torch's, else the system one). A communicator of nranks ranks from a
 * 128-byte unique id made by rank 0 (gann_nccl_unique_id) and shared by the
 * caller; gann_exchange_nccl wraps it (ncclSend/ncclRecv groups on the
 * index's stream). */
int gann_nccl_unique_id(void* id128);
int gann_nccl_comm_init(const void* id128, uint32_t rank, uint32_t nranks, int device, void** comm);
int gann_nccl_comm_destroy(void* comm);
int gann_exchange_nccl(void* comm, uint32_t rank, uint32_t nranks, gann_exchange* out);

/* Checked builds (compiled with -DGANN_CHECKED; tools/build_variant.sh):
 * the kernels test the index bounds of their shared-memory and output writes
 * on the device. Reports the largest source line of a failed check since the
 * last call (0: none) and whether this library is a checked build. */
int gann_debug_check(int device, uint32_t* failed_line, int* checked_build);

/* ---- counters (roofline) ----------------------------------------------------
 * Totals accumulated by the kernels since the last reset. */
typedef struct gann_stats {
  uint64_t queries;         /* searches run (queries + build inserts) */
  uint64_t expansions;      /* sum |V| */
  uint64_t evaluations;     /* distance evaluations by the search kernel */
  uint64_t filter_drops;    /* visited-filter inserts that did not fit */
  uint64_t adj_entries;     /* sum over expanded v of deg(v) */
  uint64_t prune_lists;     /* alpha_prune calls (insert + back-edge) */
  uint64_t prune_candidates;/* sum of prune list lengths */
  uint64_t prune_evals;     /* distances evaluated inside alpha_prune */
  uint64_t back_pairs;      /* reverse pairs grouped */
  uint64_t back_groups;     /* distinct targets */
  uint64_t back_pruned;     /* targets re-pruned */
  double build_ms[6];       /* start, search, prune, group, merge, reprune */
  uint64_t merges;          /* search: expansions whose candidates changed the beam */
  uint64_t survivors;       /* search: candidates inserted into the beam */
  uint64_t moved;           /* search: beam entries shifted by those inserts */
  uint64_t duplicates;      /* search: re-evaluated ids found already in the beam */
  uint64_t guess_hits;      /* search: expansions whose row was prefetched by a right guess */
} gann_stats;
int gann_get_stats(const gann_index* idx, gann_stats* out);
/* Frees the build's batch scratch (sized for the largest batch: ~10 GB at 10M
 * points). gann_build keeps it for the next build unless device memory is
 * tight; the next build reallocates it. */
int gann_release_scratch(gann_index* idx);
int gann_reset_stats(gann_index* idx);  /* waits for all work queued on the device first */

/* Device pointers of the resident index (points: padded rows of `stride`
 * bytes; adj: n*R uint32). For in-process callers that move the index with
 * NCCL; not needed for ordinary use. */
int gann_index_device_ptrs(const gann_index* idx, void** points, uint64_t* stride,
                           uint32_t** adj);

#ifdef __cplusplus
}
#endif
#endif /* GANN_H */
