// C++ drop-in check: the reference's own hand instances through include/gann.hpp
// (proj/tests/test_search.cpp:53-62, test_prune.cpp:38-56, test_semisort.cpp:87-113,
// test_diskann.cpp:106-120). Built by tests/cpp/Makefile; run on a GPU box.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <set>

#include "gann.hpp"

#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      std::exit(1);                                                \
    }                                                              \
  } while (0)

int main() {
  using namespace gann;
  // path graph 0-1-2-3-4 on the line, walk from 0 toward 4.2
  {
    float pts[5] = {0, 1, 2, 3, 4};
    Index idx(pts, 5, 1, ElemKind::f32, Metric::l2_squared, 2);
    HostGraph g;
    g.n = 5;
    g.capacity = 2;
    g.start = 0;
    g.adj.assign(10, GANN_NONE);
    for (uint32_t i = 0; i < 5; i++) {
      uint32_t k = 0;
      if (i > 0) g.adj[i * 2 + k++] = i - 1;
      if (i + 1 < 5) g.adj[i * 2 + k++] = i + 1;
    }
    idx.import_graph(g);
    float q = 4.2f;
    auto r = idx.search(&q, 1, SearchParams{2, 1, 0.0f}, true);
    CHECK(r[0].neighbors.size() == 1 && r[0].neighbors[0].id == 4);
    CHECK(r[0].visited.size() == 5);
    for (uint32_t i = 0; i < 5; i++) CHECK(r[0].visited[i].id == i);
    bool threw = false;
    try {
      idx.search(&q, 1, SearchParams{2, 3, 0.0f});
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  // alpha_prune on the line: p at 0, candidates 1, 2, 4
  {
    float pts[4] = {0, 1, 2, 4};
    Index idx(pts, 4, 1, ElemKind::f32, Metric::l2_squared, 3);
    std::vector<Neighbor> c = {{1, 1.0f}, {2, 4.0f}, {3, 16.0f}};
    CHECK((alpha_prune(idx, 0, c, PruneParams{3, 1.0f, PruneRule::scale_candidate}) == std::vector<uint32_t>{1}));
    CHECK((alpha_prune(idx, 0, c, PruneParams{3, 2.0f, PruneRule::scale_candidate}) == std::vector<uint32_t>{1, 3}));
  }
  // semisort: one key repeated keeps input order
  {
    std::vector<std::pair<uint32_t, uint32_t>> in;
    for (uint32_t i = 0; i < 100; i++) in.push_back({3, i});
    auto g = group_by_key(in);
    CHECK(g.groups() == 1);
    for (uint32_t i = 0; i < 100; i++) CHECK(g.pairs[i].second == i);
    CHECK((batch_ranges(10) == std::vector<std::pair<uint32_t, uint32_t>>{{1, 2}, {2, 4}, {4, 8}, {8, 10}}));
  }
  // a small u8 build keeps the invariants
  {
    const uint32_t n = 3000, d = 32;
    std::mt19937_64 rng(5);
    std::vector<uint8_t> pts(size_t(n) * d);
    for (auto& x : pts) x = static_cast<uint8_t>(rng() % 256);
    Index idx = build_diskann(pts.data(), n, d, ElemKind::u8, Metric::l2_squared, DiskannParams{16, 32, 1.2f});
    HostGraph g = idx.export_graph();
    double mean = 0;
    for (uint32_t v = 0; v < n; v++) {
      CHECK(g.degree[v] <= 16);
      std::set<uint32_t> s;
      for (uint32_t t = 0; t < g.degree[v]; t++) {
        const uint32_t u = g.out_neighbors(v)[t];
        CHECK(u < n && u != v);
        s.insert(u);
      }
      CHECK(s.size() == g.degree[v]);
      mean += g.degree[v];
    }
    CHECK(mean / n > 2.0);
    // self-queries on uniform data: an ANN search should find most points themselves
    auto r = beam_search(idx, pts.data(), 20, SearchParams{64, 10, 0.0f});
    uint32_t self = 0;
    for (uint32_t q = 0; q < 20; q++) {
      CHECK(r[q].neighbors.size() == 10);
      for (size_t t = 1; t < 10; t++) CHECK(!neighbor_less(r[q].neighbors[t], r[q].neighbors[t - 1]));
      self += r[q].neighbors[0].id == q && r[q].neighbors[0].dist == 0.0f;
    }
    CHECK(self >= 16);
  }
  std::printf("gann.hpp drop-in: ok\n");
  return 0;
}
