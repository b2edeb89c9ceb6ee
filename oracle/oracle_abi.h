/* TEST INFRASTRUCTURE — not part of the product.
 *
 * Shared C signatures of the two CPU oracles that the parity tests, smoke()
 * and bench.py's cpu_baseline leg use as checkers:
 *
 *   orc_*  oracle/gann_oracle.cpp — a scalar restatement of the reference's
 *          hot path (every function cites the reference file:line it follows)
 *   ref_*  oracle/ref_shim.cpp    — a thin extern "C" shim over the reference's
 *          own sources (proj/src/<file>.cpp under /root/reference), compiled by
 *          oracle/Makefile into oracle/_ref/ (never copied into the repo)
 *
 * Conventions (identical for both prefixes):
 *   elem   0 = u8, 1 = i8, 2 = f32          (graphann::ElemKind, core.hpp:23)
 *   metric 0 = squared L2, 1 = negated IP    (graphann::Metric, metric.hpp:13)
 *   rule   0 = scale_candidate, 1 = scale_selected (prune.hpp:19)
 *   Graphs are flat n*R uint32 rows; unused slots hold 0xFFFFFFFF and the
 *   degree of a row is the length of its non-sentinel prefix.
 *   Return codes: 0 ok, 1 invalid argument, 2 io/format, 3 internal.
 */
#ifndef GANN_ORACLE_ABI_H
#define GANN_ORACLE_ABI_H
#include <stdint.h>

#define ORACLE_DECLS(P)                                                                        \
  const char* P##last_error(void);                                                            \
  float P##distance(const void* a, const void* b, uint32_t d, int elem, int metric);          \
  int P##beam_search(const uint32_t* adj, uint32_t n, uint32_t R, uint32_t start,             \
                     const void* data, uint32_t d, int elem, int metric,                      \
                     const void* queries, uint32_t nq, uint32_t L, uint32_t k, float eps,     \
                     int visited_mode, const uint32_t* start_override, uint32_t* ids,         \
                     float* dists, uint32_t* n_visited, uint64_t* dist_comps,                 \
                     uint32_t* vis_ids, float* vis_dists, uint32_t vcap, int workers);        \
  int P##alpha_prune(uint32_t p, const uint32_t* ids, const float* dists, uint32_t m,         \
                     const void* data, uint32_t n, uint32_t d, int elem, int metric,          \
                     uint32_t R, float alpha, int rule, uint32_t* out, uint32_t* n_out,       \
                     uint64_t* dist_comps);                                                   \
  int P##group_by_key(const uint32_t* keys, const uint32_t* vals, uint64_t m, int workers,    \
                      uint32_t* out_keys, uint32_t* out_vals, uint64_t* offsets,              \
                      uint64_t* n_groups);                                                    \
  int P##choose_start(const void* data, uint32_t n, uint32_t d, int elem, int metric,         \
                      int workers, uint32_t* start);                                          \
  void P##shuffled_order(uint32_t n, uint64_t seed, uint32_t front, uint32_t* out);           \
  uint32_t P##batch_ranges(uint32_t n, uint32_t cap, uint32_t* lo, uint32_t* hi,              \
                           uint32_t max_ranges);                                              \
  int P##insert_point(uint32_t* adj, uint32_t n, uint32_t R, uint32_t start,                  \
                      const void* data, uint32_t d, int elem, int metric, uint32_t j,         \
                      uint32_t L, float alpha, int rule, uint32_t* back_targets,              \
                      uint32_t* n_back);                                                      \
  int P##apply_back_edges(uint32_t* adj, uint32_t n, uint32_t R, const void* data,            \
                          uint32_t d, int elem, int metric, const uint32_t* targets,          \
                          const uint32_t* sources, uint64_t m, float alpha, int rule,         \
                          int workers);                                                       \
  int P##build(const void* data, uint32_t n, uint32_t d, int elem, int metric, uint32_t R,    \
               uint32_t L, float alpha, int rule, uint64_t seed, uint32_t cap, int workers,   \
               uint32_t* adj, uint32_t* start);                                               \
  int P##groundtruth(const void* data, uint32_t n, const void* queries, uint32_t nq,          \
                     uint32_t d, int elem, int metric, uint32_t k, uint32_t* ids,             \
                     float* dists, int workers);                                              \
  int P##time_search(const uint32_t* adj, uint32_t n, uint32_t R, uint32_t start,              \
                     const void* data, uint32_t d, int elem, int metric, const void* queries,  \
                     uint32_t nq, uint32_t L, uint32_t k, float eps, uint32_t k_out,           \
                     int workers, uint32_t reps, double min_seconds, uint32_t* ids,            \
                     double* best_seconds, uint32_t* reps_done);                               \
  int P##range_search(const uint32_t* adj, uint32_t n, uint32_t R, uint32_t start,             \
                      const void* data, uint32_t d, int elem, int metric, const void* queries, \
                      uint32_t nq, float radius, uint32_t L, float eps, uint32_t cap,          \
                      uint32_t* counts, uint32_t* ids, float* dists);                          \
  int P##save_graph(const uint32_t* adj, uint32_t n, uint32_t R, uint32_t start,               \
                    const char* path);                                                         \
  int P##load_graph(const char* path, uint32_t* n, uint32_t* cap, uint32_t* start,             \
                    uint32_t* adj, uint64_t adj_words);                                        \
  double P##recall(const uint32_t* truth_ids, const float* truth_dists, uint32_t depth,       \
                   const uint32_t* result, uint32_t n_result, uint32_t k);

#ifdef __cplusplus
extern "C" {
#endif
ORACLE_DECLS(orc_)
ORACLE_DECLS(ref_)
/* reference only: graphann::write_vectors (src/dataset.cpp:124-140); format 0 = bin, 1 = vecs */
int ref_write_vectors(const void* data, uint32_t n, uint32_t d, int elem, const char* path, int format);
/* reference only: graphann::build_hnsw / search_hnsw (src/hnsw.cpp) behind a handle */
int ref_hnsw_build(const void* data, uint32_t n, uint32_t d, int elem, int metric, uint32_t m, uint32_t ef,
                   float alpha, int rule, uint64_t seed, int single_layer, int workers, uint32_t* handle,
                   uint32_t* num_layers, uint32_t* entry);
int ref_hnsw_export(uint32_t handle, uint32_t cap, uint32_t* levels, uint32_t* caps, uint32_t* adj);
int ref_hnsw_search(uint32_t handle, const void* data, uint32_t n, uint32_t d, int elem, int metric,
                    const void* queries, uint32_t nq, uint32_t L, uint32_t k, float eps, uint32_t* ids,
                    float* dists, uint32_t* n_visited, uint64_t* dist_comps, uint32_t* vis_ids,
                    uint32_t vcap, int workers);
void ref_hnsw_free(uint32_t handle);
/* reference only: graphann::pareto_frontier / write_csv (src/eval.cpp:205-254) on given rows */
int ref_pareto(uint32_t nrows, const uint32_t* beams, const uint32_t* ks, const float* eps, const double* recall,
               const double* qps, const double* lat, const double* dc, uint32_t* n_out, uint32_t* beams_o,
               uint32_t* ks_o, float* eps_o, double* recall_o, double* qps_o);
int ref_write_csv(const char* algorithm, const char* dataset, uint32_t n, double build_seconds, uint64_t threads,
                  uint32_t nrows, const uint32_t* beams, const uint32_t* ks, const float* eps, const double* recall,
                  const double* qps, const double* lat, const double* dc, const char* path);
#ifdef __cplusplus
}
#endif
#endif
