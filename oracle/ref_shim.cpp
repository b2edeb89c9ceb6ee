// TEST INFRASTRUCTURE — extern "C" shim over the reference's own sources.
//
// oracle/Makefile compiles this file together with the reference's hot-path
// sources where they lie (/root/reference/proj/src/*.cpp, never copied) into
// oracle/_ref/libgraphann_ref.so. Only tests/, smoke() and bench.py's
// cpu_baseline / --impl reference leg load it. Each entry point calls the
// reference's public API unchanged:
//   ref_beam_search      graphann::beam_search        (src/search.cpp:62)
//   ref_alpha_prune      graphann::alpha_prune        (src/prune.cpp:8)
//   ref_group_by_key     graphann::group_by_key       (src/semisort.cpp:15)
//   ref_choose_start     graphann::choose_start       (src/builder_common.cpp:58)
//   ref_shuffled_order   graphann::shuffled_order     (src/builder_common.cpp:99)
//   ref_batch_ranges     graphann::batch_ranges       (src/builder_common.cpp:13) + cap
//   ref_insert_point     graphann::insert_point       (src/diskann.cpp:12)
//   ref_apply_back_edges graphann::apply_back_edges   (src/builder_common.cpp:109)
//   ref_build            graphann::build_diskann      (src/diskann.cpp:31) when cap == 0,
//                        otherwise the same loop over capped ranges through the
//                        public API
//   ref_groundtruth      graphann::compute_groundtruth (src/dataset.cpp:172)
//   ref_recall           graphann::recall_k_at_n      (src/eval.cpp:14)
//   ref_hnsw_build       graphann::build_hnsw         (src/hnsw.cpp; kept behind a handle)
//   ref_hnsw_export      the handle's levels / entry / layer graphs as flat arrays
//   ref_hnsw_search      graphann::search_hnsw        (src/hnsw.cpp:130-147)
//   ref_pareto           graphann::pareto_frontier    (src/eval.cpp:205-225)
//   ref_write_csv        graphann::write_csv          (src/eval.cpp:236-254)
#include <chrono>
#include <cstdio>
#include <sstream>
#include <cstring>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "graphann/builder_common.hpp"
#include "graphann/dataset.hpp"
#include "graphann/diskann.hpp"
#include "graphann/eval.hpp"
#include "graphann/graph.hpp"
#include "graphann/hnsw.hpp"
#include "graphann/parallel.hpp"
#include "graphann/prune.hpp"
#include "graphann/search.hpp"
#include "graphann/semisort.hpp"
#include "oracle_abi.h"

using namespace graphann;

namespace {

constexpr uint32_t kSent = 0xFFFFFFFFu;
thread_local std::string g_err;

ElemKind kind(int e) { return e == 0 ? ElemKind::u8 : e == 1 ? ElemKind::i8 : ElemKind::f32; }
Metric met(int m) { return m == 0 ? Metric::l2_squared : Metric::neg_inner_product; }
PruneRule rul(int r) { return r == 0 ? PruneRule::scale_candidate : PruneRule::scale_selected; }

VectorDataset make_ds(const void* data, uint32_t n, uint32_t d, int elem) {
  VectorDataset ds(n, d, kind(elem));
  if (n) std::memcpy(ds.data(), data, ds.bytes());
  return ds;
}

NeighborGraph make_graph(const uint32_t* adj, uint32_t n, uint32_t R, uint32_t start) {
  NeighborGraph g(n, R);
  std::vector<uint32_t> row;
  for (uint32_t v = 0; v < n; v++) {
    row.clear();
    const uint32_t* r = adj + static_cast<size_t>(v) * R;
    for (uint32_t t = 0; t < R && r[t] != kSent; t++) row.push_back(r[t]);
    g.set_neighbors(v, row);
  }
  if (n) g.set_start(start);
  return g;
}

void export_graph(const NeighborGraph& g, uint32_t* adj) {
  const uint32_t R = g.capacity();
  for (uint32_t v = 0; v < g.size(); v++) {
    auto nb = g.out_neighbors(v);
    uint32_t* r = adj + static_cast<size_t>(v) * R;
    for (uint32_t t = 0; t < R; t++) r[t] = t < nb.size() ? nb[t] : kSent;
  }
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const io_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

float ref_distance(const void* a, const void* b, uint32_t d, int elem, int metric) {
  DistanceCounter c;
  return BoundMetric(met(metric), kind(elem), d)(static_cast<const std::byte*>(a),
                                                 static_cast<const std::byte*>(b), c);
}

int ref_beam_search(const uint32_t* adj, uint32_t n, uint32_t R, uint32_t start,
                    const void* data, uint32_t d, int elem, int metric, const void* queries,
                    uint32_t nq, uint32_t L, uint32_t k, float eps, int /*visited_mode*/,
                    const uint32_t* start_override, uint32_t* ids, float* dists,
                    uint32_t* n_visited, uint64_t* dist_comps, uint32_t* vis_ids,
                    float* vis_dists, uint32_t vcap, int workers) {
  return guarded([&] {
    VectorDataset ds = make_ds(data, n, d, elem);
    NeighborGraph g = make_graph(adj, n, R, start);
    const size_t stride = ds.stride();
    const std::byte* qb = static_cast<const std::byte*>(queries);
    SearchParams sp{L, k, eps};
    // the eval harness's thread boundary: parallel_for over queries (src/eval.cpp:72)
    parallel_for(nq, static_cast<size_t>(workers < 0 ? 0 : workers), [&](size_t qi, size_t) {
      VectorView q{qb + qi * stride, d, kind(elem)};
      std::optional<uint32_t> so;
      if (start_override) so = start_override[qi];
      SearchResult r = beam_search(g, ds, met(metric), q, sp, nullptr, so);
      for (uint32_t t = 0; t < k; t++) {
        bool have = t < r.neighbors.size();
        ids[qi * k + t] = have ? r.neighbors[t].id : kSent;
        dists[qi * k + t] = have ? r.neighbors[t].dist : std::numeric_limits<float>::infinity();
      }
      n_visited[qi] = static_cast<uint32_t>(r.visited.size());
      if (dist_comps) dist_comps[qi] = r.dist_comps;
      if (vis_ids)
        for (uint32_t t = 0; t < vcap && t < r.visited.size(); t++) {
          vis_ids[qi * vcap + t] = r.visited[t].id;
          vis_dists[qi * vcap + t] = r.visited[t].dist;
        }
    });
  });
}

int ref_alpha_prune(uint32_t p, const uint32_t* ids, const float* dists, uint32_t m,
                    const void* data, uint32_t n, uint32_t d, int elem, int metric, uint32_t R,
                    float alpha, int rule, uint32_t* out, uint32_t* n_out, uint64_t* dist_comps) {
  return guarded([&] {
    VectorDataset ds = make_ds(data, n, d, elem);
    std::vector<Neighbor> c(m);
    for (uint32_t i = 0; i < m; i++) c[i] = {ids[i], dists[i]};
    DistanceCounter cnt;
    auto r = alpha_prune(p, c, PruneParams{R, alpha, rul(rule)}, ds, met(metric), cnt);
    std::copy(r.begin(), r.end(), out);
    *n_out = static_cast<uint32_t>(r.size());
    if (dist_comps) *dist_comps = cnt.count;
  });
}

int ref_group_by_key(const uint32_t* keys, const uint32_t* vals, uint64_t m, int workers,
                     uint32_t* out_keys, uint32_t* out_vals, uint64_t* offsets,
                     uint64_t* n_groups) {
  return guarded([&] {
    std::vector<std::pair<uint32_t, uint32_t>> in(m);
    for (uint64_t i = 0; i < m; i++) in[i] = {keys[i], vals[i]};
    GroupedPairs gp = group_by_key(in, static_cast<size_t>(workers < 0 ? 0 : workers));
    for (uint64_t i = 0; i < m; i++) {
      out_keys[i] = gp.pairs[i].first;
      out_vals[i] = gp.pairs[i].second;
    }
    for (size_t i = 0; i < gp.group_offsets.size(); i++) offsets[i] = gp.group_offsets[i];
    *n_groups = gp.groups();
  });
}

int ref_choose_start(const void* data, uint32_t n, uint32_t d, int elem, int metric,
                     int workers, uint32_t* start) {
  return guarded([&] {
    VectorDataset ds = make_ds(data, n, d, elem);
    *start = choose_start(ds, met(metric), static_cast<size_t>(workers < 0 ? 0 : workers));
  });
}

void ref_shuffled_order(uint32_t n, uint64_t seed, uint32_t front, uint32_t* out) {
  auto o = shuffled_order(n, seed, front);
  std::copy(o.begin(), o.end(), out);
}

uint32_t ref_batch_ranges(uint32_t n, uint32_t cap, uint32_t* lo, uint32_t* hi,
                          uint32_t max_ranges) {
  std::vector<std::pair<uint32_t, uint32_t>> r;
  if (cap == 0) {
    r = batch_ranges(n);
  } else {  // hi = min(2*lo, lo + cap, n) — SURVEY.md §B.3 item 3 (probe 3)
    for (uint64_t a = 1; a < n;) {
      uint64_t h = std::min<uint64_t>({a << 1, a + cap, n});
      r.emplace_back(static_cast<uint32_t>(a), static_cast<uint32_t>(h));
      a = h;
    }
  }
  for (size_t i = 0; i < r.size() && i < max_ranges; i++) {
    lo[i] = r[i].first;
    hi[i] = r[i].second;
  }
  return static_cast<uint32_t>(r.size());
}

int ref_insert_point(uint32_t* adj, uint32_t n, uint32_t R, uint32_t start, const void* data,
                     uint32_t d, int elem, int metric, uint32_t j, uint32_t L, float alpha,
                     int rule, uint32_t* back_targets, uint32_t* n_back) {
  return guarded([&] {
    VectorDataset ds = make_ds(data, n, d, elem);
    NeighborGraph g = make_graph(adj, n, R, start);
    DiskannParams p;
    p.degree_bound = R;
    p.build_beam = L;
    p.alpha = alpha;
    p.rule = rul(rule);
    DistanceCounter c;
    auto back = insert_point(g, ds, met(metric), j, p, c);
    for (size_t i = 0; i < back.size(); i++) back_targets[i] = back[i].first;
    *n_back = static_cast<uint32_t>(back.size());
    export_graph(g, adj);
  });
}

int ref_apply_back_edges(uint32_t* adj, uint32_t n, uint32_t R, const void* data, uint32_t d,
                         int elem, int metric, const uint32_t* targets, const uint32_t* sources,
                         uint64_t m, float alpha, int rule, int workers) {
  return guarded([&] {
    VectorDataset ds = make_ds(data, n, d, elem);
    NeighborGraph g = make_graph(adj, n, R, 0);
    std::vector<std::pair<uint32_t, uint32_t>> e(m);
    for (uint64_t i = 0; i < m; i++) e[i] = {targets[i], sources[i]};
    size_t w = resolve_workers(static_cast<size_t>(workers < 0 ? 0 : workers));
    std::vector<DistanceCounter> counters(w);
    apply_back_edges(g, ds, met(metric), e, PruneParams{R, alpha, rul(rule)}, w, counters);
    export_graph(g, adj);
  });
}

int ref_build(const void* data, uint32_t n, uint32_t d, int elem, int metric, uint32_t R,
              uint32_t L, float alpha, int rule, uint64_t seed, uint32_t cap, int workers,
              uint32_t* adj, uint32_t* start) {
  return guarded([&] {
    VectorDataset ds = make_ds(data, n, d, elem);
    DiskannParams p;
    p.degree_bound = R;
    p.build_beam = L;
    p.alpha = alpha;
    p.rule = rul(rule);
    p.seed = seed;
    const size_t w = static_cast<size_t>(workers < 0 ? 0 : workers);
    if (cap == 0) {
      NeighborGraph g = build_diskann(ds, met(metric), p, w);
      export_graph(g, adj);
      *start = g.start();
      return;
    }
    // Capped schedule through the reference's public API (the loop of
    // src/diskann.cpp:44-69 driven by capped ranges).
    if (n == 0) throw std::invalid_argument("cannot build over an empty dataset");
    NeighborGraph g(n, R);
    uint32_t s = choose_start(ds, met(metric), w);
    g.set_start(s);
    auto order = shuffled_order(n, mix64(seed, 0x696e73657274ULL), s);
    size_t rw = resolve_workers(w);
    std::vector<DistanceCounter> counters(rw);
    PruneParams pp{R, alpha, rul(rule)};
    for (uint64_t lo = 1; lo < n;) {
      uint64_t hi = std::min<uint64_t>({lo << 1, lo + cap, n});
      const uint32_t count = static_cast<uint32_t>(hi - lo);
      std::vector<std::vector<std::pair<uint32_t, uint32_t>>> back(count);
      parallel_for(count, w, [&](size_t b, size_t worker) {
        back[b] = insert_point(g, ds, met(metric), order[lo + b], p, counters[worker]);
      });
      std::vector<std::pair<uint32_t, uint32_t>> edges;
      for (const auto& v : back) edges.insert(edges.end(), v.begin(), v.end());
      apply_back_edges(g, ds, met(metric), edges, pp, w, counters);
      lo = hi;
    }
    export_graph(g, adj);
    *start = g.start();
  });
}

int ref_groundtruth(const void* data, uint32_t n, const void* queries, uint32_t nq, uint32_t d,
                    int elem, int metric, uint32_t k, uint32_t* ids, float* dists, int workers) {
  return guarded([&] {
    VectorDataset ds = make_ds(data, n, d, elem);
    VectorDataset qs = make_ds(queries, nq, d, elem);
    GroundTruth gt =
        compute_groundtruth(ds, qs, k, met(metric), static_cast<size_t>(workers < 0 ? 0 : workers));
    std::copy(gt.ids.begin(), gt.ids.end(), ids);
    std::copy(gt.dists.begin(), gt.dists.end(), dists);
  });
}

// measure_qps (src/eval.cpp:57-101): parallel_for over the queries, best of
// `reps` passes (at least `reps`, continuing until min_seconds of work).
int ref_time_search(const uint32_t* adj, uint32_t n, uint32_t R, uint32_t start, const void* data,
                    uint32_t d, int elem, int metric, const void* queries, uint32_t nq, uint32_t L,
                    uint32_t k, float eps, uint32_t k_out, int workers, uint32_t reps,
                    double min_seconds, uint32_t* ids, double* best_seconds, uint32_t* reps_done) {
  return guarded([&] {
    VectorDataset ds = make_ds(data, n, d, elem);
    NeighborGraph g = make_graph(adj, n, R, start);
    const size_t stride = ds.stride();
    const std::byte* qb = static_cast<const std::byte*>(queries);
    SearchParams sp{L, k, eps};
    double best = 1e300, total = 0.0;
    uint32_t r = 0;
    for (; r < reps || total < min_seconds; r++) {
      auto t0 = std::chrono::steady_clock::now();
      parallel_for(nq, static_cast<size_t>(workers < 0 ? 0 : workers), [&](size_t qi, size_t) {
        VectorView q{qb + qi * stride, d, kind(elem)};
        SearchResult res = beam_search(g, ds, met(metric), q, sp);
        if (r == 0 && ids)
          for (uint32_t t = 0; t < k_out; t++)
            ids[qi * k_out + t] = t < res.neighbors.size() ? res.neighbors[t].id : kSent;
      });
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      best = std::min(best, s);
      total += s;
      if (r >= 1000) break;
    }
    *best_seconds = best;
    if (reps_done) *reps_done = r;
  });
}

// graphann::range_search (src/search.cpp:133-149)
int ref_range_search(const uint32_t* adj, uint32_t n, uint32_t R, uint32_t start, const void* data,
                     uint32_t d, int elem, int metric, const void* queries, uint32_t nq, float radius,
                     uint32_t L, float eps, uint32_t cap, uint32_t* counts, uint32_t* ids, float* dists) {
  return guarded([&] {
    VectorDataset ds = make_ds(data, n, d, elem);
    NeighborGraph g = make_graph(adj, n, R, start);
    const std::byte* qb = static_cast<const std::byte*>(queries);
    for (uint32_t qi = 0; qi < nq; qi++) {
      VectorView q{qb + size_t(qi) * ds.stride(), d, kind(elem)};
      RangeResult r = range_search(g, ds, met(metric), q, radius, SearchParams{L, 1, eps});
      counts[qi] = static_cast<uint32_t>(r.in_range.size());
      for (uint32_t t = 0; t < cap; t++) {
        const bool have = t < r.in_range.size();
        ids[size_t(qi) * cap + t] = have ? r.in_range[t].id : kSent;
        dists[size_t(qi) * cap + t] = have ? r.in_range[t].dist : std::numeric_limits<float>::infinity();
      }
    }
  });
}

// graphann::save_graph / load_graph (src/graph.cpp:101-178)
int ref_save_graph(const uint32_t* adj, uint32_t n, uint32_t R, uint32_t start, const char* path) {
  return guarded([&] { save_graph(make_graph(adj, n, R, start), std::string(path)); });
}

int ref_load_graph(const char* path, uint32_t* n, uint32_t* cap, uint32_t* start, uint32_t* adj,
                   uint64_t adj_words) {
  return guarded([&] {
    NeighborGraph g = load_graph(std::string(path));
    *n = g.size();
    *cap = g.capacity();
    *start = g.start();
    if (adj && adj_words >= uint64_t(g.size()) * g.capacity()) export_graph(g, adj);
  });
}

int ref_write_vectors(const void* data, uint32_t n, uint32_t d, int elem, const char* path, int format) {
  return guarded([&] {
    write_vectors(make_ds(data, n, d, elem), std::string(path), format == 0 ? FileFormat::bin : FileFormat::vecs);
  });
}

double ref_recall(const uint32_t* truth_ids, const float* truth_dists, uint32_t depth,
                  const uint32_t* result, uint32_t n_result, uint32_t k) {
  try {
    return recall_k_at_n(std::span<const uint32_t>(truth_ids, depth),
                         std::span<const float>(truth_dists, depth),
                         std::span<const uint32_t>(result, n_result), k);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

// ---- layered (HNSW) search: the reference's own builder and search_hnsw ----
// The built HnswIndex stays inside the shim (its members are private to the
// reference's build/load functions); tests export its layers for the GPU.
static std::vector<std::unique_ptr<HnswIndex>> g_hnsw;

int ref_hnsw_build(const void* data, uint32_t n, uint32_t d, int elem, int metric, uint32_t m,
                   uint32_t ef, float alpha, int rule, uint64_t seed, int single_layer, int workers,
                   uint32_t* handle, uint32_t* num_layers, uint32_t* entry) {
  return guarded([&] {
    VectorDataset ds = make_ds(data, n, d, elem);
    HnswParams p;
    p.m = m;
    p.ef_construction = ef;
    p.alpha = alpha;
    p.rule = rul(rule);
    p.seed = seed;
    p.single_layer = single_layer != 0;
    g_hnsw.push_back(std::make_unique<HnswIndex>(
        build_hnsw(ds, met(metric), p, static_cast<size_t>(workers < 0 ? 0 : workers))));
    const HnswIndex& h = *g_hnsw.back();
    *handle = static_cast<uint32_t>(g_hnsw.size() - 1);
    *num_layers = h.num_layers();
    *entry = h.entry();
  });
}

// levels[n]; adj holds layer l's rows at (l * n + v) * cap, cap >= every layer's capacity
int ref_hnsw_export(uint32_t handle, uint32_t cap, uint32_t* levels, uint32_t* caps, uint32_t* adj) {
  return guarded([&] {
    if (handle >= g_hnsw.size() || !g_hnsw[handle]) throw std::invalid_argument("bad hnsw handle");
    const HnswIndex& h = *g_hnsw[handle];
    const uint32_t n = h.size();
    for (uint32_t v = 0; v < n; v++) levels[v] = h.level(v);
    for (uint32_t l = 0; l < h.num_layers(); l++) {
      const NeighborGraph& g = h.layer(l);
      if (g.capacity() > cap) throw std::invalid_argument("layer capacity above cap");
      caps[l] = g.capacity();
      for (uint32_t v = 0; v < n; v++) {
        auto nb = g.out_neighbors(v);
        uint32_t* r = adj + (static_cast<size_t>(l) * n + v) * cap;
        for (uint32_t t = 0; t < cap; t++) r[t] = t < nb.size() ? nb[t] : kSent;
      }
    }
  });
}

int ref_hnsw_search(uint32_t handle, const void* data, uint32_t n, uint32_t d, int elem, int metric,
                    const void* queries, uint32_t nq, uint32_t L, uint32_t k, float eps, uint32_t* ids,
                    float* dists, uint32_t* n_visited, uint64_t* dist_comps, uint32_t* vis_ids,
                    uint32_t vcap, int workers) {
  return guarded([&] {
    if (handle >= g_hnsw.size() || !g_hnsw[handle]) throw std::invalid_argument("bad hnsw handle");
    const HnswIndex& h = *g_hnsw[handle];
    VectorDataset ds = make_ds(data, n, d, elem);
    const size_t stride = ds.stride();
    const std::byte* qb = static_cast<const std::byte*>(queries);
    SearchParams sp{L, k, eps};
    parallel_for(nq, static_cast<size_t>(workers < 0 ? 0 : workers), [&](size_t qi, size_t) {
      VectorView q{qb + qi * stride, d, kind(elem)};
      SearchResult r = search_hnsw(h, ds, met(metric), q, sp, nullptr);
      for (uint32_t t = 0; t < k; t++) {
        bool have = t < r.neighbors.size();
        ids[qi * k + t] = have ? r.neighbors[t].id : kSent;
        dists[qi * k + t] = have ? r.neighbors[t].dist : std::numeric_limits<float>::infinity();
      }
      n_visited[qi] = static_cast<uint32_t>(r.visited.size());
      if (dist_comps) dist_comps[qi] = r.dist_comps;
      if (vis_ids)
        for (uint32_t t = 0; t < vcap && t < r.visited.size(); t++) vis_ids[qi * vcap + t] = r.visited[t].id;
    });
  });
}

void ref_hnsw_free(uint32_t handle) {
  if (handle < g_hnsw.size()) g_hnsw[handle].reset();
}

// ---- eval harness: pareto_frontier / write_csv on caller-given rows ----------
static std::vector<EvalRow> rows_of(uint32_t nrows, const uint32_t* beams, const uint32_t* ks, const float* eps,
                                    const double* recall, const double* qps, const double* lat, const double* dc) {
  std::vector<EvalRow> rows(nrows);
  for (uint32_t i = 0; i < nrows; i++) rows[i] = {beams[i], ks[i], eps[i], recall[i], qps[i], lat[i], dc[i]};
  return rows;
}

int ref_pareto(uint32_t nrows, const uint32_t* beams, const uint32_t* ks, const float* eps, const double* recall,
               const double* qps, const double* lat, const double* dc, uint32_t* n_out, uint32_t* beams_o,
               uint32_t* ks_o, float* eps_o, double* recall_o, double* qps_o) {
  return guarded([&] {
    std::vector<EvalRow> rows = rows_of(nrows, beams, ks, eps, recall, qps, lat, dc);
    std::vector<EvalRow> f = pareto_frontier(rows);
    *n_out = static_cast<uint32_t>(f.size());
    for (size_t i = 0; i < f.size(); i++) {
      beams_o[i] = f[i].beam;
      ks_o[i] = f[i].k;
      eps_o[i] = f[i].epsilon;
      recall_o[i] = f[i].recall;
      qps_o[i] = f[i].qps;
    }
  });
}

int ref_write_csv(const char* algorithm, const char* dataset, uint32_t n, double build_seconds, uint64_t threads,
                  uint32_t nrows, const uint32_t* beams, const uint32_t* ks, const float* eps, const double* recall,
                  const double* qps, const double* lat, const double* dc, const char* path) {
  return guarded([&] {
    EvalReport r;
    r.meta.algorithm = algorithm;
    r.meta.dataset = dataset;
    r.meta.n = n;
    r.meta.build_seconds = build_seconds;
    r.meta.threads = threads;
    r.rows = rows_of(nrows, beams, ks, eps, recall, qps, lat, dc);
    // the stream overload (src/eval.cpp:236-245) into memory, then plain stdio:
    // the path overload's std::ofstream crashes inside a process that has
    // loaded numpy's bundled runtime libraries
    std::ostringstream os;
    write_csv(r, os);
    const std::string text = os.str();
    FILE* f = std::fopen(path, "wb");
    if (!f) throw io_error(std::string("cannot open for writing: ") + path);
    const size_t wrote = std::fwrite(text.data(), 1, text.size(), f);
    std::fclose(f);
    if (wrote != text.size()) throw io_error(std::string("write failed: ") + path);
  });
}

}  // extern "C"
