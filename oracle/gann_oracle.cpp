// TEST INFRASTRUCTURE — CPU restatement of the reference's hot path.
//
// This file is the parity checker for the B200 kernels, not the product. Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg
// may load it. It restates, in plain scalar C++, the behaviour of graphann
// (/root/reference/proj) on the Vamana batch-build + beam-search path. Every
// function names the reference file:line it follows. The restatement is pinned
// against the reference itself: tests/test_oracle_cpu.py compares it with the
// compiled reference (oracle/_ref, built by oracle/Makefile from the reference
// sources) and with the golden fixtures under tests/golden/ that
// tests/golden/make_golden.py generated from that same compiled reference.
//
// Third-party arithmetic: the insertion order depends on libstdc++'s
// std::mt19937_64 + std::shuffle (builder_common.cpp:99-107); this file calls
// the same library (GCC 13.3 libstdc++ in this image) rather than re-deriving
// it.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "oracle_abi.h"

namespace {

constexpr uint32_t kSent = 0xFFFFFFFFu;
constexpr float kInf = std::numeric_limits<float>::infinity();
thread_local std::string g_err;

struct Nb {
  uint32_t id;
  float dist;
};

// neighbor_less: (dist, id) lexicographic — include/graphann/core.hpp:42-44.
inline bool nb_less(const Nb& a, const Nb& b) {
  return a.dist < b.dist || (a.dist == b.dist && a.id < b.id);
}

// splitmix64 finaliser and its 2-argument fold — include/graphann/core.hpp:47-58.
inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline uint64_t mix64(uint64_t a, uint64_t b) { return mix64(a ^ mix64(b)); }

inline size_t esize(int elem) { return elem == 2 ? 4 : 1; }

// Distance kernels — src/metric.cpp:38-59. Integer kinds accumulate in int32
// and cast once; f32 accumulates sequentially in float with separate multiply
// and add (the reference is built without -march, so no FMA contraction; this
// file is compiled with -ffp-contract=off to keep that).
template <typename T, typename Acc>
float l2sq(const void* a, const void* b, uint32_t d) {
  const T* x = static_cast<const T*>(a);
  const T* y = static_cast<const T*>(b);
  Acc acc = 0;
  for (uint32_t i = 0; i < d; i++) {
    Acc diff = static_cast<Acc>(x[i]) - static_cast<Acc>(y[i]);
    acc += diff * diff;
  }
  return static_cast<float>(acc);
}
template <typename T, typename Acc>
float negip(const void* a, const void* b, uint32_t d) {
  const T* x = static_cast<const T*>(a);
  const T* y = static_cast<const T*>(b);
  Acc acc = 0;
  for (uint32_t i = 0; i < d; i++) acc += static_cast<Acc>(x[i]) * static_cast<Acc>(y[i]);
  return -static_cast<float>(acc);
}

float dist_fn(const void* a, const void* b, uint32_t d, int elem, int metric) {
  if (metric == 0) {
    if (elem == 0) return l2sq<uint8_t, int32_t>(a, b, d);
    if (elem == 1) return l2sq<int8_t, int32_t>(a, b, d);
    return l2sq<float, float>(a, b, d);
  }
  if (elem == 0) return negip<uint8_t, int32_t>(a, b, d);
  if (elem == 1) return negip<int8_t, int32_t>(a, b, d);
  return negip<float, float>(a, b, d);
}

struct Data {
  const uint8_t* base;
  uint32_t n, d;
  int elem, metric;
  size_t stride;
  const uint8_t* row(uint32_t i) const { return base + static_cast<size_t>(i) * stride; }
  float operator()(const void* a, const void* b, uint64_t& cnt) const {
    cnt++;
    return dist_fn(a, b, d, elem, metric);
  }
};

struct Graph {
  uint32_t* adj;
  uint32_t n, R;
  uint32_t degree(uint32_t v) const {
    const uint32_t* r = adj + static_cast<size_t>(v) * R;
    uint32_t k = 0;
    while (k < R && r[k] != kSent) k++;
    return k;
  }
  const uint32_t* row(uint32_t v) const { return adj + static_cast<size_t>(v) * R; }
  // set_neighbors — src/graph.cpp:42-59 (bound, range and self-loop checks).
  void set(uint32_t v, const std::vector<uint32_t>& ids) {
    if (ids.size() > R) throw std::invalid_argument("degree exceeds capacity");
    uint32_t* r = adj + static_cast<size_t>(v) * R;
    for (size_t i = 0; i < ids.size(); i++) {
      if (ids[i] >= n) throw std::invalid_argument("neighbor id out of range");
      if (ids[i] == v) throw std::invalid_argument("self loop");
      r[i] = ids[i];
    }
    for (size_t i = ids.size(); i < R; i++) r[i] = kSent;
  }
};

template <typename F>
void run_parallel(size_t n, int workers, F&& f) {
  size_t w = workers <= 0 ? std::max(1u, std::thread::hardware_concurrency())
                          : static_cast<size_t>(workers);
  if (w > n) w = n;
  if (w <= 1) {
    for (size_t i = 0; i < n; i++) f(i);
    return;
  }
  std::atomic<size_t> cur{0};
  std::vector<std::thread> ts;
  std::exception_ptr err;
  std::atomic<bool> claimed{false};
  for (size_t t = 0; t < w; t++) {
    ts.emplace_back([&] {
      try {
        for (size_t i; (i = cur.fetch_add(1)) < n;) f(i);
      } catch (...) {
        if (!claimed.exchange(true)) err = std::current_exception();
        cur.store(n);
      }
    });
  }
  for (auto& t : ts) t.join();
  if (err) std::rethrow_exception(err);
}

// search_seed — src/search.cpp:52-58.
uint64_t search_seed(const uint8_t* q, uint32_t dim, int elem, uint32_t start) {
  uint64_t h = mix64(start, dim);
  size_t take = std::min<size_t>(16, static_cast<size_t>(dim) * esize(elem));
  uint64_t buf[2] = {0, 0};
  std::memcpy(buf, q, take);
  return mix64(h ^ buf[0], buf[1]);
}

struct SearchOut {
  std::vector<Nb> neighbors, visited;
  uint64_t dist_comps = 0;
};

// beam_search — src/search.cpp:62-131 (validation :32-48). visited_mode 0
// uses an exact seen-set; mode 1 reproduces ApproxVisitedSet
// (include/graphann/search.hpp:24-38: beam*beam slots, mix64(id ^ seed) % slots,
// overwrite on collision) so dist_comps matches the reference as well.
SearchOut beam_search(const Graph& g, const Data& ds, const uint8_t* q, uint32_t L, uint32_t k,
                      float eps, int mode, uint32_t start) {
  SearchOut res;
  if (g.n == 0) return res;
  if (start >= g.n) throw std::invalid_argument("start vertex out of range");
  struct Entry {
    float dist;
    uint32_t id;
    bool expanded;
  };
  auto less = [](const Entry& a, const Entry& b) {
    return a.dist < b.dist || (a.dist == b.dist && a.id < b.id);
  };
  std::vector<Entry> beam;
  beam.reserve(L + 1);
  std::unordered_set<uint32_t> exact_seen;
  std::vector<uint32_t> table;
  uint64_t seed = 0;
  if (mode == 1) {
    table.assign(static_cast<size_t>(L) * L, kSent);
    seed = search_seed(q, ds.d, ds.elem, start);
  }
  auto slot = [&](uint32_t id) { return static_cast<size_t>(mix64(id ^ seed) % table.size()); };
  auto seen_contains = [&](uint32_t id) {
    return mode == 1 ? table[slot(id)] == id : exact_seen.count(id) != 0;
  };
  auto seen_insert = [&](uint32_t id) {
    if (mode == 1)
      table[slot(id)] = id;
    else
      exact_seen.insert(id);
  };
  // push — src/search.cpp:83-90: sorted insert, exact (dist,id) duplicates
  // dropped, anything past position L falls off.
  auto push = [&](uint32_t id, float dist) {
    Entry e{dist, id, false};
    auto it = std::lower_bound(beam.begin(), beam.end(), e, less);
    if (it != beam.end() && it->id == id && it->dist == dist) return;
    if (beam.size() >= L && it == beam.end()) return;
    beam.insert(it, e);
    if (beam.size() > L) beam.pop_back();
  };
  push(start, ds(q, ds.row(start), res.dist_comps));  // :92-93
  seen_insert(start);
  std::unordered_set<uint32_t> expanded;
  while (true) {  // :95-122
    size_t next = beam.size();
    for (size_t i = 0; i < beam.size(); i++)
      if (!beam[i].expanded) {
        next = i;
        break;
      }
    if (next == beam.size()) break;
    // k-gate with epsilon slack — :105-107
    float best_k = beam.size() >= k ? beam[k - 1].dist : kInf;
    float limit = best_k == kInf ? kInf : best_k + eps * std::fabs(best_k);
    if (beam[next].dist > limit) break;
    beam[next].expanded = true;
    uint32_t cur = beam[next].id;
    float cd = beam[next].dist;
    if (!expanded.insert(cur).second) continue;  // :113
    res.visited.push_back({cur, cd});
    const uint32_t* nbrs = g.row(cur);
    for (uint32_t t = 0; t < g.R && nbrs[t] != kSent; t++) {  // :117-121
      uint32_t nb = nbrs[t];
      if (seen_contains(nb)) continue;
      seen_insert(nb);
      push(nb, ds(q, ds.row(nb), res.dist_comps));
    }
  }
  res.neighbors = res.visited;  // :124-126
  std::sort(res.neighbors.begin(), res.neighbors.end(), nb_less);
  if (res.neighbors.size() > k) res.neighbors.resize(k);
  return res;
}

// alpha_prune — src/prune.cpp:8-44.
std::vector<uint32_t> alpha_prune(uint32_t p, const std::vector<Nb>& candidates, uint32_t R,
                                  float alpha, int rule, const Data& ds, uint64_t& cnt) {
  if (R == 0) throw std::invalid_argument("degree bound must be positive");
  if (!(alpha > 0.0f)) throw std::invalid_argument("alpha must be positive");
  std::vector<Nb> cand;
  for (const auto& c : candidates)
    if (c.id != p) cand.push_back(c);
  std::sort(cand.begin(), cand.end(), nb_less);
  std::vector<uint32_t> out;
  std::vector<char> culled(cand.size(), 0);
  for (size_t i = 0; i < cand.size() && out.size() < R; i++) {
    if (culled[i]) continue;
    const Nb sel = cand[i];
    out.push_back(sel.id);
    if (out.size() == R) break;
    if (sel.dist == 0.0f) continue;  // :32 zero-distance picks cull nothing
    for (size_t j = i + 1; j < cand.size(); j++) {
      if (culled[j]) continue;
      float via = ds(ds.row(sel.id), ds.row(cand[j].id), cnt);
      // one IEEE f32 multiply, never contracted (prune.cpp:37-39)
      bool drop = rule == 0 ? alpha * via <= cand[j].dist : via < alpha * sel.dist;
      if (drop) culled[j] = 1;
    }
  }
  return out;
}

// group_by_key — src/semisort.cpp:15-73. The reference's output order is a
// pure function of the input: buckets bit_ceil(max(1, m/1024)) by
// mix64(key) & mask, each bucket sorted by (key, input index). Restated as one
// sort on (bucket, key, index).
void group_by_key(const uint32_t* keys, const uint32_t* vals, uint64_t m, uint32_t* ok,
                  uint32_t* ov, uint64_t* offsets, uint64_t* ng) {
  if (m == 0) {
    *ng = 0;
    return;
  }
  uint64_t nb = 1;
  while (nb < std::max<uint64_t>(1, m / 1024)) nb <<= 1;
  const uint64_t mask = nb - 1;
  std::vector<uint64_t> idx(m);
  for (uint64_t i = 0; i < m; i++) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
    uint64_t ba = mix64(keys[a]) & mask, bb = mix64(keys[b]) & mask;
    if (ba != bb) return ba < bb;
    if (keys[a] != keys[b]) return keys[a] < keys[b];
    return a < b;
  });
  uint64_t g = 0;
  for (uint64_t i = 0; i < m; i++) {
    ok[i] = keys[idx[i]];
    ov[i] = vals[idx[i]];
    if (i == 0 || ok[i] != ok[i - 1]) offsets[g++] = i;
  }
  offsets[g] = m;
  *ng = g;
}

// choose_start — src/builder_common.cpp:58-97: double column sums, float
// centroid, sequential float distance (no FMA), argmin by (dist, id).
uint32_t choose_start(const Data& ds) {
  if (ds.n == 0) throw std::invalid_argument("cannot pick a start point of an empty dataset");
  std::vector<double> sum(ds.d, 0.0);
  for (uint32_t i = 0; i < ds.n; i++) {
    const uint8_t* r = ds.row(i);
    for (uint32_t j = 0; j < ds.d; j++) {
      double x = ds.elem == 0   ? static_cast<double>(r[j])
                 : ds.elem == 1 ? static_cast<double>(reinterpret_cast<const int8_t*>(r)[j])
                                : static_cast<double>(reinterpret_cast<const float*>(r)[j]);
      sum[j] += x;
    }
  }
  std::vector<float> c(ds.d);
  for (uint32_t j = 0; j < ds.d; j++) c[j] = static_cast<float>(sum[j] / ds.n);
  Nb best{0, kInf};
  for (uint32_t i = 0; i < ds.n; i++) {
    const uint8_t* r = ds.row(i);
    float acc = 0.0f;
    for (uint32_t j = 0; j < ds.d; j++) {
      float x = ds.elem == 0   ? static_cast<float>(r[j])
                : ds.elem == 1 ? static_cast<float>(reinterpret_cast<const int8_t*>(r)[j])
                               : reinterpret_cast<const float*>(r)[j];
      if (ds.metric == 0) {
        float diff = x - c[j];
        acc += diff * diff;
      } else {
        acc += x * c[j];
      }
    }
    float dist = ds.metric == 0 ? acc : -acc;
    Nb cand{i, dist};
    if (nb_less(cand, best)) best = cand;
  }
  return best.id;
}

// shuffled_order — src/builder_common.cpp:99-107.
std::vector<uint32_t> shuffled_order(uint32_t n, uint64_t seed, uint32_t front) {
  std::vector<uint32_t> order(n);
  for (uint32_t i = 0; i < n; i++) order[i] = i;
  std::mt19937_64 rng(seed);
  std::shuffle(order.begin(), order.end(), rng);
  auto it = std::find(order.begin(), order.end(), front);
  std::iter_swap(order.begin(), it);
  return order;
}

// batch_ranges — src/builder_common.cpp:13-20 ([1,2),[2,4),... clipped to n).
// cap > 0 adds the BASELINE config-0 batch cap as hi = min(2*lo, lo + cap, n)
// (the schedule SURVEY.md §B.3 item 3 / probe 3 uses).
std::vector<std::pair<uint32_t, uint32_t>> batch_ranges(uint32_t n, uint32_t cap) {
  std::vector<std::pair<uint32_t, uint32_t>> r;
  for (uint64_t lo = 1; lo < n;) {
    uint64_t hi = std::min<uint64_t>(lo << 1, n);
    if (cap > 0) hi = std::min<uint64_t>(hi, lo + cap);
    r.emplace_back(static_cast<uint32_t>(lo), static_cast<uint32_t>(hi));
    lo = hi;
  }
  return r;
}

// insert_point — src/diskann.cpp:12-29: drained search {L, L, 0}, prune the
// visited list, write the out-list, return the reverse pairs (q, j).
std::vector<uint32_t> insert_point(Graph& g, const Data& ds, uint32_t j, uint32_t start,
                                   uint32_t L, float alpha, int rule, uint64_t& cnt) {
  SearchOut s = beam_search(g, ds, ds.row(j), L, L, 0.0f, 0, start);
  cnt += s.dist_comps;
  std::vector<uint32_t> kept = alpha_prune(j, s.visited, g.R, alpha, rule, ds, cnt);
  g.set(j, kept);
  return kept;
}

// apply_back_edges — src/builder_common.cpp:109-140: group by target (input
// order kept inside a group), append new sources (first occurrence wins),
// re-prune with fresh distances when the list exceeds R.
void apply_back_edges(Graph& g, const Data& ds, const uint32_t* targets, const uint32_t* sources,
                      uint64_t m, float alpha, int rule, int workers) {
  if (m == 0) return;
  std::vector<uint32_t> gk(m), gv(m);
  std::vector<uint64_t> off(m + 1);
  uint64_t ng = 0;
  group_by_key(targets, sources, m, gk.data(), gv.data(), off.data(), &ng);
  run_parallel(ng, workers, [&](size_t gi) {
    uint64_t cnt = 0;
    const uint32_t t = gk[off[gi]];
    std::vector<uint32_t> merged(g.row(t), g.row(t) + g.degree(t));
    for (uint64_t e = off[gi]; e < off[gi + 1]; e++)
      if (std::find(merged.begin(), merged.end(), gv[e]) == merged.end()) merged.push_back(gv[e]);
    if (merged.size() <= g.R) {
      g.set(t, merged);
      return;
    }
    std::vector<Nb> c;
    for (uint32_t id : merged) c.push_back({id, ds(ds.row(t), ds.row(id), cnt)});
    g.set(t, alpha_prune(t, c, g.R, alpha, rule, ds, cnt));
  });
}

// build_diskann — src/diskann.cpp:31-70 (with the optional batch cap above).
uint32_t build(Graph& g, const Data& ds, uint32_t L, float alpha, int rule, uint64_t seed,
               uint32_t cap, int workers) {
  if (ds.n == 0) throw std::invalid_argument("cannot build over an empty dataset");
  if (L == 0 || g.R == 0) throw std::invalid_argument("build beam and degree bound must be positive");
  std::fill(g.adj, g.adj + static_cast<size_t>(g.n) * g.R, kSent);
  uint32_t start = choose_start(ds);
  std::vector<uint32_t> order = shuffled_order(ds.n, mix64(seed, 0x696e73657274ULL), start);
  for (auto [lo, hi] : batch_ranges(ds.n, cap)) {
    std::vector<std::vector<uint32_t>> back(hi - lo);
    run_parallel(hi - lo, workers, [&](size_t b) {
      uint64_t cnt = 0;
      back[b] = insert_point(g, ds, order[lo + b], start, L, alpha, rule, cnt);
    });
    std::vector<uint32_t> tg, src;
    for (uint32_t b = 0; b < hi - lo; b++)
      for (uint32_t q : back[b]) {
        tg.push_back(q);
        src.push_back(order[lo + b]);
      }
    apply_back_edges(g, ds, tg.data(), src.data(), tg.size(), alpha, rule, workers);
  }
  return start;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

float orc_distance(const void* a, const void* b, uint32_t d, int elem, int metric) {
  return dist_fn(a, b, d, elem, metric);
}

int orc_beam_search(const uint32_t* adj, uint32_t n, uint32_t R, uint32_t start,
                    const void* data, uint32_t d, int elem, int metric, const void* queries,
                    uint32_t nq, uint32_t L, uint32_t k, float eps, int visited_mode,
                    const uint32_t* start_override, uint32_t* ids, float* dists,
                    uint32_t* n_visited, uint64_t* dist_comps, uint32_t* vis_ids,
                    float* vis_dists, uint32_t vcap, int workers) {
  return guarded([&] {
    // validate_search_args — src/search.cpp:32-48
    if (L == 0 || k == 0) throw std::invalid_argument("beam and k must be positive");
    if (k > L) throw std::invalid_argument("k exceeds beam");
    if (!(eps >= 0.0f && eps <= 0.25f)) throw std::invalid_argument("epsilon must lie in [0, 0.25]");
    Graph g{const_cast<uint32_t*>(adj), n, R};
    Data ds{static_cast<const uint8_t*>(data), n, d, elem, metric, d * esize(elem)};
    const uint8_t* qb = static_cast<const uint8_t*>(queries);
    run_parallel(nq, workers, [&](size_t qi) {
      uint32_t s = start_override ? start_override[qi] : start;
      SearchOut r = beam_search(g, ds, qb + qi * ds.stride, L, k, eps, visited_mode, s);
      for (uint32_t t = 0; t < k; t++) {
        bool have = t < r.neighbors.size();
        ids[qi * k + t] = have ? r.neighbors[t].id : kSent;
        dists[qi * k + t] = have ? r.neighbors[t].dist : kInf;
      }
      n_visited[qi] = static_cast<uint32_t>(r.visited.size());
      if (dist_comps) dist_comps[qi] = r.dist_comps;
      if (vis_ids)
        for (uint32_t t = 0; t < vcap && t < r.visited.size(); t++) {
          vis_ids[static_cast<size_t>(qi) * vcap + t] = r.visited[t].id;
          vis_dists[static_cast<size_t>(qi) * vcap + t] = r.visited[t].dist;
        }
    });
  });
}

int orc_alpha_prune(uint32_t p, const uint32_t* ids, const float* dists, uint32_t m,
                    const void* data, uint32_t n, uint32_t d, int elem, int metric, uint32_t R,
                    float alpha, int rule, uint32_t* out, uint32_t* n_out, uint64_t* dist_comps) {
  return guarded([&] {
    Data ds{static_cast<const uint8_t*>(data), n, d, elem, metric, d * esize(elem)};
    std::vector<Nb> c(m);
    for (uint32_t i = 0; i < m; i++) c[i] = {ids[i], dists[i]};
    uint64_t cnt = 0;
    auto r = alpha_prune(p, c, R, alpha, rule, ds, cnt);
    std::copy(r.begin(), r.end(), out);
    *n_out = static_cast<uint32_t>(r.size());
    if (dist_comps) *dist_comps = cnt;
  });
}

int orc_group_by_key(const uint32_t* keys, const uint32_t* vals, uint64_t m, int,
                     uint32_t* out_keys, uint32_t* out_vals, uint64_t* offsets,
                     uint64_t* n_groups) {
  return guarded([&] { group_by_key(keys, vals, m, out_keys, out_vals, offsets, n_groups); });
}

int orc_choose_start(const void* data, uint32_t n, uint32_t d, int elem, int metric, int,
                     uint32_t* start) {
  return guarded([&] {
    Data ds{static_cast<const uint8_t*>(data), n, d, elem, metric, d * esize(elem)};
    *start = choose_start(ds);
  });
}

void orc_shuffled_order(uint32_t n, uint64_t seed, uint32_t front, uint32_t* out) {
  auto o = shuffled_order(n, seed, front);
  std::copy(o.begin(), o.end(), out);
}

uint32_t orc_batch_ranges(uint32_t n, uint32_t cap, uint32_t* lo, uint32_t* hi,
                          uint32_t max_ranges) {
  auto r = batch_ranges(n, cap);
  for (size_t i = 0; i < r.size() && i < max_ranges; i++) {
    lo[i] = r[i].first;
    hi[i] = r[i].second;
  }
  return static_cast<uint32_t>(r.size());
}

int orc_insert_point(uint32_t* adj, uint32_t n, uint32_t R, uint32_t start, const void* data,
                     uint32_t d, int elem, int metric, uint32_t j, uint32_t L, float alpha,
                     int rule, uint32_t* back_targets, uint32_t* n_back) {
  return guarded([&] {
    Graph g{adj, n, R};
    Data ds{static_cast<const uint8_t*>(data), n, d, elem, metric, d * esize(elem)};
    uint64_t cnt = 0;
    auto kept = insert_point(g, ds, j, start, L, alpha, rule, cnt);
    std::copy(kept.begin(), kept.end(), back_targets);
    *n_back = static_cast<uint32_t>(kept.size());
  });
}

int orc_apply_back_edges(uint32_t* adj, uint32_t n, uint32_t R, const void* data, uint32_t d,
                         int elem, int metric, const uint32_t* targets, const uint32_t* sources,
                         uint64_t m, float alpha, int rule, int workers) {
  return guarded([&] {
    Graph g{adj, n, R};
    Data ds{static_cast<const uint8_t*>(data), n, d, elem, metric, d * esize(elem)};
    apply_back_edges(g, ds, targets, sources, m, alpha, rule, workers);
  });
}

int orc_build(const void* data, uint32_t n, uint32_t d, int elem, int metric, uint32_t R,
              uint32_t L, float alpha, int rule, uint64_t seed, uint32_t cap, int workers,
              uint32_t* adj, uint32_t* start) {
  return guarded([&] {
    Graph g{adj, n, R};
    Data ds{static_cast<const uint8_t*>(data), n, d, elem, metric, d * esize(elem)};
    *start = build(g, ds, L, alpha, rule, seed, cap, workers);
  });
}

// compute_groundtruth — src/dataset.cpp:172-217: exact top-k by (dist, id).
int orc_groundtruth(const void* data, uint32_t n, const void* queries, uint32_t nq, uint32_t d,
                    int elem, int metric, uint32_t k, uint32_t* ids, float* dists, int workers) {
  return guarded([&] {
    if (k == 0 || k > n) throw std::invalid_argument("groundtruth: bad k");
    Data ds{static_cast<const uint8_t*>(data), n, d, elem, metric, d * esize(elem)};
    const uint8_t* qb = static_cast<const uint8_t*>(queries);
    run_parallel(nq, workers, [&](size_t qi) {
      std::vector<Nb> all(n);
      uint64_t cnt = 0;
      for (uint32_t i = 0; i < n; i++) all[i] = {i, ds(qb + qi * ds.stride, ds.row(i), cnt)};
      std::partial_sort(all.begin(), all.begin() + k, all.end(), nb_less);
      for (uint32_t t = 0; t < k; t++) {
        ids[qi * k + t] = all[t].id;
        dists[qi * k + t] = all[t].dist;
      }
    });
  });
}

// measure_qps (src/eval.cpp:57-101) restated: threads over queries, best of reps.
int orc_time_search(const uint32_t* adj, uint32_t n, uint32_t R, uint32_t start, const void* data,
                    uint32_t d, int elem, int metric, const void* queries, uint32_t nq, uint32_t L,
                    uint32_t k, float eps, uint32_t k_out, int workers, uint32_t reps,
                    double min_seconds, uint32_t* ids, double* best_seconds, uint32_t* reps_done) {
  return guarded([&] {
    Graph g{const_cast<uint32_t*>(adj), n, R};
    Data ds{static_cast<const uint8_t*>(data), n, d, elem, metric, d * esize(elem)};
    const uint8_t* qb = static_cast<const uint8_t*>(queries);
    double best = 1e300, total = 0.0;
    uint32_t r = 0;
    for (; r < reps || total < min_seconds; r++) {
      auto t0 = std::chrono::steady_clock::now();
      run_parallel(nq, workers, [&](size_t qi) {
        SearchOut res = beam_search(g, ds, qb + qi * ds.stride, L, k, eps, 0, start);
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

// range_search — src/search.cpp:133-149: drain {L, L, eps}, keep visited with
// dist <= internal_radius (src/dataset.cpp:248-250), sorted by (dist, id).
int orc_range_search(const uint32_t* adj, uint32_t n, uint32_t R, uint32_t start, const void* data,
                     uint32_t d, int elem, int metric, const void* queries, uint32_t nq, float radius,
                     uint32_t L, float eps, uint32_t cap, uint32_t* counts, uint32_t* ids, float* dists) {
  return guarded([&] {
    if (!(radius > 0)) throw std::invalid_argument("range radius must be positive");
    Graph g{const_cast<uint32_t*>(adj), n, R};
    Data ds{static_cast<const uint8_t*>(data), n, d, elem, metric, d * esize(elem)};
    const float rr = metric == 0 ? radius * radius : radius;
    const uint8_t* qb = static_cast<const uint8_t*>(queries);
    for (uint32_t qi = 0; qi < nq; qi++) {
      SearchOut r = beam_search(g, ds, qb + qi * ds.stride, L, L, eps, 0, start);
      std::vector<Nb> in;
      for (const auto& v : r.visited)
        if (v.dist <= rr) in.push_back(v);
      std::sort(in.begin(), in.end(), nb_less);
      counts[qi] = static_cast<uint32_t>(in.size());
      for (uint32_t t = 0; t < cap; t++) {
        const bool have = t < in.size();
        ids[size_t(qi) * cap + t] = have ? in[t].id : kSent;
        dists[size_t(qi) * cap + t] = have ? in[t].dist : kInf;
      }
    }
  });
}

// ANNG layout — src/graph.cpp:101-178
int orc_save_graph(const uint32_t* adj, uint32_t n, uint32_t R, uint32_t start, const char* path) {
  return guarded([&] {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot open for writing");
    Graph g{const_cast<uint32_t*>(adj), n, R};
    out.write("ANNG", 4);
    const uint32_t h[4] = {1u, n, R, start};
    out.write(reinterpret_cast<const char*>(h), sizeof(h));
    std::vector<uint32_t> deg(n);
    for (uint32_t v = 0; v < n; v++) deg[v] = g.degree(v);
    out.write(reinterpret_cast<const char*>(deg.data()), std::streamsize(n) * 4);
    for (uint32_t v = 0; v < n; v++) out.write(reinterpret_cast<const char*>(g.row(v)), std::streamsize(deg[v]) * 4);
  });
}

int orc_load_graph(const char* path, uint32_t* n, uint32_t* cap, uint32_t* start, uint32_t* adj,
                   uint64_t adj_words) {
  return guarded([&] {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open for reading");
    char magic[4];
    uint32_t h[4];
    in.read(magic, 4);
    in.read(reinterpret_cast<char*>(h), sizeof(h));
    if (!in || std::memcmp(magic, "ANNG", 4) != 0 || h[0] != 1u) throw std::runtime_error("not a graph file");
    *n = h[1];
    *cap = h[2];
    *start = h[3];
    if (!adj || adj_words < uint64_t(h[1]) * h[2]) return;
    std::vector<uint32_t> deg(h[1]);
    in.read(reinterpret_cast<char*>(deg.data()), std::streamsize(h[1]) * 4);
    std::fill(adj, adj + uint64_t(h[1]) * h[2], kSent);
    for (uint32_t v = 0; v < h[1]; v++) in.read(reinterpret_cast<char*>(adj + uint64_t(v) * h[2]), std::streamsize(deg[v]) * 4);
    if (!in) throw std::runtime_error("truncated graph data");
  });
}

// recall_k_at_n — src/eval.cpp:14-33: ties with the k-th truth distance count.
double orc_recall(const uint32_t* truth_ids, const float* truth_dists, uint32_t depth,
                  const uint32_t* result, uint32_t n_result, uint32_t k) {
  if (k == 0 || depth < k) return -1.0;
  const float kth = truth_dists[k - 1];
  uint32_t matched = 0;
  for (uint32_t r = 0; r < n_result; r++) {
    bool hit = false;
    for (uint32_t j = 0; j < k && !hit; j++) hit = truth_ids[j] == result[r];
    for (uint32_t j = k; j < depth && !hit && truth_dists[j] == kth; j++)
      hit = truth_ids[j] == result[r];
    if (hit) matched++;
  }
  return static_cast<double>(std::min(matched, k)) / k;
}

}  // extern "C"
