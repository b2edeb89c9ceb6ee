// gann.hpp — header-only C++ mirror of graphann's hot-path API over the C ABI.
//
// A graphann user swaps `#include "graphann/diskann.hpp"` / `search.hpp` for
// this header and links libgann_b200.so. Names, parameter structs, argument
// meaning and error behaviour follow the reference:
//   DiskannParams            include/graphann/diskann.hpp:14-20
//   SearchParams             include/graphann/search.hpp:14-18
//   PruneParams / PruneRule  include/graphann/prune.hpp:19-24
//   Neighbor, neighbor_less  include/graphann/core.hpp:37-44
//   build_diskann            include/graphann/diskann.hpp:36-37
//   beam_search              include/graphann/search.hpp:57-60 (batched here)
//   alpha_prune              include/graphann/prune.hpp:31-33
//   group_by_key             include/graphann/semisort.hpp:21-22
//   choose_start / shuffled_order / batch_ranges / apply_back_edges
//                            include/graphann/builder_common.hpp:17-34
//   insert_point             include/graphann/diskann.hpp:26-29
// std::invalid_argument is thrown where the reference throws it (GANN_EINVAL);
// CUDA failures throw gann::cuda_error. The graph lives in HBM inside Index;
// export_graph() returns the reference's flat fixed-degree layout.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gann.h"

namespace gann {

class cuda_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class io_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == GANN_OK) return;
  const std::string msg = gann_last_error();
  if (rc == GANN_EINVAL) throw std::invalid_argument(msg);
  if (rc == GANN_EIO) throw io_error(msg);
  throw cuda_error(msg);
}

enum class ElemKind : int { u8 = GANN_U8, i8 = GANN_I8, f32 = GANN_F32 };
enum class Metric : int { l2_squared = GANN_L2, neg_inner_product = GANN_IP };
enum class PruneRule : int { scale_candidate = GANN_SCALE_CANDIDATE, scale_selected = GANN_SCALE_SELECTED };

struct Neighbor {
  uint32_t id = 0;
  float dist = 0.0f;
};
inline bool neighbor_less(const Neighbor& a, const Neighbor& b) {
  return a.dist < b.dist || (a.dist == b.dist && a.id < b.id);
}

struct DiskannParams {
  uint32_t degree_bound = 64;  // R
  uint32_t build_beam = 128;   // L
  float alpha = 1.2f;
  PruneRule rule = PruneRule::scale_candidate;
  uint64_t seed = 42;
  uint32_t max_batch = 0;      // 0 = the reference's uncapped prefix doubling
};
struct SearchParams {
  uint32_t beam = 10;
  uint32_t k = 10;
  float epsilon = 0.0f;
};
struct PruneParams {
  uint32_t degree_bound = 64;
  float alpha = 1.2f;
  PruneRule rule = PruneRule::scale_candidate;
};

// Per-query result of a batched search (graphann::SearchResult).
struct SearchResult {
  std::vector<Neighbor> neighbors;  // k best of visited, ascending (dist, id)
  std::vector<Neighbor> visited;    // expansion order (filled when requested)
  uint64_t dist_comps = 0;
};

// Flat host copy of a graph: n rows of `capacity` ids, GANN_NONE padded.
struct HostGraph {
  uint32_t n = 0, capacity = 0, start = 0;
  std::vector<uint32_t> adj;
  std::vector<uint32_t> degree;
  const uint32_t* out_neighbors(uint32_t v) const { return adj.data() + size_t(v) * capacity; }
};

// Points + graph resident in HBM (graphann::VectorDataset + NeighborGraph).
class Index {
 public:
  Index(const void* points, uint64_t n, uint32_t d, ElemKind elem, Metric metric,
        uint32_t degree_bound, int device = 0)
      : d_(d), elem_(elem), metric_(metric) {
    gann_index* h = nullptr;
    check(gann_index_create(points, n, d, static_cast<int>(elem), static_cast<int>(metric),
                            degree_bound, device, &h));
    h_.reset(h);
  }
  gann_index* handle() const { return h_.get(); }
  uint32_t dim() const { return d_; }

  void build(const DiskannParams& p) {
    check(gann_build(h_.get(), p.build_beam, p.alpha, static_cast<int>(p.rule), p.seed, p.max_batch));
  }
  void import_graph(const HostGraph& g) { check(gann_import_graph(h_.get(), g.adj.data(), g.start)); }
  void release_scratch() { check(gann_release_scratch(h_.get())); }
  HostGraph export_graph() const {
    uint64_t n = 0;
    uint32_t R = 0, start = 0;
    check(gann_index_info(h_.get(), &n, nullptr, nullptr, nullptr, &R, &start));
    HostGraph g;
    g.n = static_cast<uint32_t>(n);
    g.capacity = R;
    g.adj.resize(size_t(n) * R);
    g.degree.resize(n);
    check(gann_export_graph(h_.get(), g.adj.data(), g.degree.data(), &g.start));
    return g;
  }

  // Batched beam_search: `queries` holds nq rows of d elements.
  std::vector<SearchResult> search(const void* queries, uint32_t nq, const SearchParams& p,
                                   bool want_visited = false,
                                   const std::vector<uint32_t>* start_override = nullptr) const {
    std::vector<uint32_t> ids(size_t(nq) * p.k), nvis(nq);
    std::vector<float> dists(size_t(nq) * p.k);
    std::vector<uint64_t> dc(nq);
    const uint32_t vcap = want_visited ? 8 * p.beam + 64 : 0;
    std::vector<uint32_t> vi(size_t(nq) * vcap);
    std::vector<float> vd(size_t(nq) * vcap);
    check(gann_search(h_.get(), queries, nq, p.k, p.beam, p.k, p.epsilon, GANN_VISITED_FAST,
                      start_override ? start_override->data() : nullptr, ids.data(), dists.data(),
                      nvis.data(), dc.data(), vcap ? vi.data() : nullptr, vcap ? vd.data() : nullptr,
                      vcap));
    std::vector<SearchResult> out(nq);
    for (uint32_t q = 0; q < nq; q++) {
      for (uint32_t t = 0; t < p.k; t++)
        if (ids[size_t(q) * p.k + t] != GANN_NONE)
          out[q].neighbors.push_back({ids[size_t(q) * p.k + t], dists[size_t(q) * p.k + t]});
      for (uint32_t t = 0; t < nvis[q] && t < vcap; t++)
        out[q].visited.push_back({vi[size_t(q) * vcap + t], vd[size_t(q) * vcap + t]});
      out[q].dist_comps = dc[q];
    }
    return out;
  }

  // Serving form (gann_search_async): enqueue one batch on `stream` (a
  // cudaStream_t) with caller scratch of search_async_scratch(nq, k) bytes;
  // h_ids / h_dists (nq*k, pinned) are valid once the stream reaches it.
  uint64_t search_async_scratch(uint32_t nq, uint32_t k) const { return gann_search_async_scratch(h_.get(), nq, k); }
  void search_async(const void* h_queries, uint32_t nq, const SearchParams& p, uint32_t* h_ids, float* h_dists,
                    void* d_scratch, uint64_t scratch_bytes, void* stream) const {
    check(gann_search_async(h_.get(), h_queries, nq, p.k, p.beam, p.k, p.epsilon, h_ids, h_dists, d_scratch,
                            scratch_bytes, stream));
  }

  uint32_t choose_start() const {
    uint32_t s = 0;
    check(gann_choose_start(h_.get(), &s));
    return s;
  }

 private:
  struct Free {
    void operator()(gann_index* p) const { gann_index_free(p); }
  };
  std::unique_ptr<gann_index, Free> h_;
  uint32_t d_;
  ElemKind elem_;
  Metric metric_;
};

// Layered index (graphann::HnswIndex): layer 0 is an Index (borrowed), the upper
// layers are graphs over the same ids, each n rows of m_upper ids.
class HnswIndex {
 public:
  HnswIndex(Index& layer0, const std::vector<HostGraph>& upper, uint32_t entry) {
    std::vector<uint32_t> flat;
    const uint32_t m = upper.empty() ? 0 : upper[0].capacity;
    for (const HostGraph& g : upper) {
      if (g.capacity != m) throw std::invalid_argument("upper layers must share one row capacity");
      flat.insert(flat.end(), g.adj.begin(), g.adj.end());
    }
    gann_hnsw* h = nullptr;
    check(gann_hnsw_create(layer0.handle(), 1 + static_cast<uint32_t>(upper.size()),
                           flat.empty() ? nullptr : flat.data(), m, entry, &h));
    h_.reset(h);
  }
  gann_hnsw* handle() const { return h_.get(); }

 private:
  struct Free {
    void operator()(gann_hnsw* p) const { gann_hnsw_free(p); }
  };
  std::unique_ptr<gann_hnsw, Free> h_;
};

// graphann::search_hnsw (src/hnsw.cpp:130-147), batched over queries.
inline std::vector<SearchResult> search_hnsw(const HnswIndex& h, const void* queries, uint32_t nq,
                                             const SearchParams& p) {
  std::vector<uint32_t> ids(size_t(nq) * p.k), nvis(nq);
  std::vector<float> dists(size_t(nq) * p.k);
  std::vector<uint64_t> dc(nq);
  check(gann_hnsw_search(h.handle(), queries, nq, p.k, p.beam, p.k, p.epsilon, GANN_VISITED_FAST, ids.data(),
                         dists.data(), nvis.data(), dc.data()));
  std::vector<SearchResult> out(nq);
  for (uint32_t q = 0; q < nq; q++) {
    for (uint32_t t = 0; t < p.k; t++)
      if (ids[size_t(q) * p.k + t] != GANN_NONE)
        out[q].neighbors.push_back({ids[size_t(q) * p.k + t], dists[size_t(q) * p.k + t]});
    out[q].dist_comps = dc[q];
  }
  return out;
}

// ---- free functions with the reference's names ------------------------------------
inline Index build_diskann(const void* points, uint64_t n, uint32_t d, ElemKind elem, Metric metric,
                           const DiskannParams& p, int device = 0) {
  if (n == 0) throw std::invalid_argument("cannot build over an empty dataset");
  Index idx(points, n, d, elem, metric, p.degree_bound, device);
  idx.build(p);
  return idx;
}

inline std::vector<SearchResult> beam_search(const Index& idx, const void* queries, uint32_t nq,
                                             const SearchParams& p) {
  return idx.search(queries, nq, p);
}

inline std::vector<uint32_t> alpha_prune(const Index& idx, uint32_t p,
                                         const std::vector<Neighbor>& candidates,
                                         const PruneParams& pp) {
  std::vector<uint32_t> ids, out(pp.degree_bound);
  std::vector<float> dists;
  for (const auto& c : candidates) {
    ids.push_back(c.id);
    dists.push_back(c.dist);
  }
  const uint64_t offs[2] = {0, ids.size()};
  uint32_t nout = 0;
  check(gann_alpha_prune(idx.handle(), &p, offs, 1, ids.data(), dists.data(), pp.alpha,
                         static_cast<int>(pp.rule), out.data(), &nout));
  out.resize(nout);
  return out;
}

struct GroupedPairs {
  std::vector<std::pair<uint32_t, uint32_t>> pairs;
  std::vector<size_t> group_offsets;
  size_t groups() const { return group_offsets.empty() ? 0 : group_offsets.size() - 1; }
};

inline GroupedPairs group_by_key(const std::vector<std::pair<uint32_t, uint32_t>>& in, int device = 0) {
  GroupedPairs g;
  const uint64_t m = in.size();
  if (m == 0) return g;
  std::vector<uint32_t> k(m), v(m), ok(m), ov(m);
  for (uint64_t i = 0; i < m; i++) {
    k[i] = in[i].first;
    v[i] = in[i].second;
  }
  std::vector<uint64_t> off(m + 1);
  uint64_t ng = 0;
  check(gann_group_by_key(k.data(), v.data(), m, device, ok.data(), ov.data(), off.data(), &ng));
  g.pairs.resize(m);
  for (uint64_t i = 0; i < m; i++) g.pairs[i] = {ok[i], ov[i]};
  g.group_offsets.assign(off.begin(), off.begin() + ng + 1);
  return g;
}

inline std::vector<uint32_t> shuffled_order(uint32_t n, uint64_t seed, uint32_t front) {
  std::vector<uint32_t> o(n);
  gann_shuffled_order(n, seed, front, o.data());
  return o;
}

inline std::vector<std::pair<uint32_t, uint32_t>> batch_ranges(uint64_t n, uint32_t max_batch = 0) {
  const uint32_t cap = 64 + (max_batch ? static_cast<uint32_t>(n / max_batch) : 0);
  std::vector<uint32_t> lo(cap), hi(cap);
  const uint32_t c = gann_batch_ranges(n, max_batch, lo.data(), hi.data(), cap);
  std::vector<std::pair<uint32_t, uint32_t>> r;
  for (uint32_t i = 0; i < c && i < cap; i++) r.emplace_back(lo[i], hi[i]);
  return r;
}

inline void apply_back_edges(Index& idx, const std::vector<std::pair<uint32_t, uint32_t>>& edges,
                             const PruneParams& pp) {
  std::vector<uint32_t> t, s;
  for (const auto& e : edges) {
    t.push_back(e.first);
    s.push_back(e.second);
  }
  check(gann_apply_back_edges(idx.handle(), t.data(), s.data(), t.size(), pp.alpha,
                              static_cast<int>(pp.rule)));
}

// insert_point for one point: returns the reverse pairs (q, j).
inline std::vector<std::pair<uint32_t, uint32_t>> insert_point(Index& idx, uint32_t j,
                                                               const DiskannParams& p) {
  uint32_t R = 0;
  check(gann_index_info(idx.handle(), nullptr, nullptr, nullptr, nullptr, &R, nullptr));
  std::vector<uint32_t> back(R);
  check(gann_insert_batch(idx.handle(), &j, 1, p.build_beam, p.alpha, static_cast<int>(p.rule),
                          back.data()));
  std::vector<std::pair<uint32_t, uint32_t>> out;
  for (uint32_t q : back)
    if (q != GANN_NONE) out.emplace_back(q, j);
  return out;
}

}  // namespace gann
