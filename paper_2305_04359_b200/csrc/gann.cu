// gann.cu — host side of the C ABI (include/gann.h): HBM-resident index,
// batch-build driver and search front end. Plain C++ + CUDA runtime; no torch.
//
// Build driver = graphann::build_diskann (src/diskann.cpp:31-70) re-planned
// for one GPU: the start vertex is chosen on the device, the insertion order
// is drawn on the host with the same libstdc++ std::mt19937_64 + std::shuffle
// call as the reference (src/builder_common.cpp:99-107), and every prefix-
// doubling batch runs as
//   search  (one warp per inserted point, drained beam {L, L, 0})
//   prune   (one CTA per point: alpha_prune of its visited list, written
//            straight into its out-row — the point is unreachable until its
//            back-edges land, src/diskann.cpp:56-59)
//   group   (count / bump-offsets / scatter of the batch's reverse pairs)
//   merge   (one CTA per target: restore pair order, append, dedupe; rows
//            that overflow R are staged with fresh distances)
//   reprune (alpha_prune of the staged rows)
// on one stream, with one host read-back per phase-2 step for grid sizes.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <random>
#include <stdexcept>
#include <string>
#include <map>
#include <mutex>
#include <set>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/gann.h"
#include "common.cuh"
#include "internal.h"

using namespace gann;

namespace {

thread_local std::string g_err;

struct Error {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(GANN_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

// gann_last_error() text for failures reported outside gann.cu
void gann::set_last_error(const std::string& msg) { g_err = msg; }

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return GANN_OK;
  } catch (const Error& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return GANN_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GANN_ECUDA;
  }
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  // Grows geometrically: cudaFree synchronises the device and large cudaMallocs
  // are slow, so a build must not reallocate on every slightly larger batch.
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (p) cudaFree(p);
    p = nullptr;
    size_t want = std::max<size_t>({bytes, cap + cap / 2, size_t(1) << 16});
    want = (want + 4095) & ~size_t(4095);
    cap = 0;
    cu(cudaMalloc(&p, want), "cudaMalloc scratch");
    cap = want;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

size_t elem_bytes(int elem) { return elem == GANN_F32 ? 4 : 1; }

uint32_t env_u32(const char* name, uint32_t dflt) {
  const char* v = std::getenv(name);
  return v && *v ? static_cast<uint32_t>(std::strtoul(v, nullptr, 10)) : dflt;
}

// Shared-memory visited table of the fast search mode: a pure performance
// knob — it trades re-evaluated rows against per-warp shared memory, i.e.
// resident warps; it never reports a false positive, so results do not
// depend on it. A slot stores the 15-bit remainder of a bijective hash of the
// id while n fits (half the bytes of an id slot, so twice the entries); a
// bucket of 4 (2, 1) slots then covers n <= 2^(log2 + 13) (+14, +15). Larger
// n store whole ids, in buckets of 4 as well.
// Past L = 1024 the table grows with the beam (GANN_HASH_PER_BEAM slots per
// beam slot, default 2). A walk of beam L evaluates ~10 L distinct ids and a
// small table re-gathers evicted rows (c1, L = 1024, 2048 slots: 3.7x the
// distinct rows), but the shared memory a larger table takes costs resident
// warps, and that costs more: measured at c1, L = 832 / 1024, 2048 slots ->
// 20.5 / 26.5 ms per 10k queries; 4, 8, 16 slots per beam slot -> 21.6 /
// 26.5, 27.5 / 34.0, 38.4 / 47.0 ms.
void hash_config(uint32_t L, uint64_t n, uint32_t* log2, uint32_t* bits, uint32_t* ways) {
  const uint32_t forced = std::min<uint32_t>(env_u32("GANN_HASH_LOG2", 0), 15);
  const bool narrow = env_u32("GANN_HASH16", 1) != 0;
  const uint64_t per_beam = env_u32("GANN_HASH_PER_BEAM", 2);
  uint32_t grow = 0;  // doublings past the base table for large beams
  if (L > 256)
    while (grow < 4 && (uint64_t(2048) << grow) < per_beam * L) grow++;
  // 512 < L <= 2048: half the table (1024 slots) leaves room for more
  // resident warps, which pays more than the re-gathers it adds (c1, L = 832:
  // 19.8 vs 20.5 ms per 10k queries; L = 1024: 25.8 vs 26.5; L = 200: 4.91 vs
  // 4.74, so small beams keep 2048)
  const uint32_t base = (L > 512 && L <= 2048) ? 10 : 11;
  uint32_t l = forced ? std::max<uint32_t>(forced, 5) : base + grow;
  // u16 remainder slots; 2-way buckets (the bucket's newest id in the low
  // half) halve the conflict evictions of a direct-mapped table of the same size
  const uint32_t w = env_u32("GANN_HASH_WAYS", 4);
  const uint32_t wl = w >= 4 ? 2 : (w == 2 ? 1 : 0);  // log2(ways)
  *ways = 1u << wl;
  while (*ways > 1 && !(narrow && n <= (uint64_t(1) << (l + 15 - (31 - __builtin_clz(*ways)))))) *ways >>= 1;
  const uint32_t b = l + 15 - (31 - __builtin_clz(*ways));
  if (narrow && n <= (uint64_t(1) << b)) {
    *log2 = l;
    *bits = b;
    return;
  }
  // u32 id slots (n above 2^26); 4-way buckets unless GANN_HASH_WAYS is 1 or 2
  // (measured at 100M, c4 generator: 1024 slots in buckets of 4 beat 512 / 2048,
  // and direct mapping, at L = 64 and 200)
  *ways = w >= 4 ? 4 : 1;
  *log2 = forced ? std::max<uint32_t>(forced, 5) : (*ways == 4 || L <= 160 ? 10 : 9) + grow;
  *bits = 0;
}

}  // namespace

// std::shuffle's swap log. libstdc++'s shuffle touches its range only through
// iter_swap(i, first + pos) for i = first + 1 .. last - 1 (bits/stl_algo.h, both
// its one-draw-two-swaps path and the plain one). Run over this iterator it
// draws from the generator exactly as over a vector, but a "swap" only records
// log[i] = pos — sequential writes instead of random ones — and the permutation
// is resolved on the device (misc.cu launch_shuffle_from_log). Same library
// call, same draws, so the order equals shuffled_order's (src/builder_common.cpp:99-107).
namespace swaplog {
struct Val {
  uint32_t src;
};
struct Ref {
  uint32_t idx;
  uint32_t* log;
  operator Val() const { return Val{idx}; }
  const Ref& operator=(const Ref& o) const {  // *a = *b inside a three-step swap: a receives b's element
    log[idx] = o.idx;
    return *this;
  }
  const Ref& operator=(const Val&) const { return *this; }  // *b = tmp: the other half of the same swap
  friend void swap(Ref a, Ref b) { a.log[a.idx] = b.idx; }
};
struct It {
  using iterator_category = std::random_access_iterator_tag;
  using value_type = Val;
  using difference_type = int64_t;
  using pointer = void;
  using reference = Ref;
  int64_t i;
  uint32_t* log;
  Ref operator*() const { return Ref{static_cast<uint32_t>(i), log}; }
  Ref operator[](difference_type k) const { return Ref{static_cast<uint32_t>(i + k), log}; }
  It& operator++() { ++i; return *this; }
  It operator++(int) { It t = *this; ++i; return t; }
  It& operator--() { --i; return *this; }
  It operator--(int) { It t = *this; --i; return t; }
  It& operator+=(difference_type k) { i += k; return *this; }
  It& operator-=(difference_type k) { i -= k; return *this; }
  friend It operator+(It a, difference_type k) { a.i += k; return a; }
  friend It operator+(difference_type k, It a) { a.i += k; return a; }
  friend It operator-(It a, difference_type k) { a.i -= k; return a; }
  friend difference_type operator-(It a, It b) { return a.i - b.i; }
  friend bool operator==(It a, It b) { return a.i == b.i; }
  friend bool operator!=(It a, It b) { return a.i != b.i; }
  friend bool operator<(It a, It b) { return a.i < b.i; }
  friend bool operator>(It a, It b) { return a.i > b.i; }
  friend bool operator<=(It a, It b) { return a.i <= b.i; }
  friend bool operator>=(It a, It b) { return a.i >= b.i; }
};
}  // namespace swaplog

// log[i] = the position std::shuffle(first, first + n, mt19937_64(seed)) swaps element i with (log[0] = 0)
static void shuffle_swap_log(uint64_t n, uint64_t seed, uint32_t* log) {
  for (uint64_t i = 0; i < n; i++) log[i] = static_cast<uint32_t>(i);
  std::mt19937_64 rng(seed);
  std::shuffle(swaplog::It{0, log}, swaplog::It{static_cast<int64_t>(n), log}, rng);
}

constexpr uint32_t kQueryCounters = 64;  // per-launch query counters per index

struct gann_index {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t n = 0;
  uint32_t d = 0;
  int elem = 0, metric = 0;
  uint32_t R = 0;
  uint32_t start = 0;
  uint32_t row_bytes = 0;
  uint64_t stride = 0;
  Geometry geom{};
  uint8_t* points = nullptr;
  uint32_t* adj = nullptr;
  uint8_t* spre = nullptr;   // per row: length of its prune-output prefix (PruneArgs::spre)
  float spre_alpha = -1.0f;  // the (alpha, rule) those prefixes were pruned with
  int spre_rule = -1;
  uint32_t* tcount = nullptr;
  uint32_t* tgroup = nullptr;
  unsigned long long* stats = nullptr;  // kStCount
  unsigned long long* counters = nullptr;  // kCntNum
  uint32_t* flags = nullptr;  // [0] overflow, [1] too_long
  uint32_t* qctr = nullptr;   // kQueryCounters per-launch query counters (round robin)
  std::atomic<uint32_t> qslot{0};
  double build_ms[6] = {0, 0, 0, 0, 0, 0};
  std::vector<std::tuple<cudaEvent_t, cudaEvent_t, int>> timers;  // recorded, not yet read
  uint64_t back_pairs = 0, back_groups = 0, back_pruned = 0;
  // scratch
  DevBuf q, qstaged, qids, qdists, qnvis, qdc, qvids, qvd, qstart, table;
  DevBuf order, vis_ids, vis_d, nvis;
  DevBuf gtarget, gcnt, goff, gcursor, gsrc, poff, plen, pid, pdist, bigg, pls, plb;
  DevBuf pt, ps, ok, ov, misc, gt, bins;
  uint32_t staged_nq = 0;
  bool staged = false;  // gann_stage_queries has run
  // vertex partitioning (1 partition = the whole graph)
  uint32_t part_rank = 0, part_count = 1, part_size = 0, part_base = 0, part_rows = 0;
  uint32_t** d_parts = nullptr;            // device table of partition row pointers
  std::vector<void*> ipc_open;             // peer partitions mapped through CUDA IPC
  // partitioned build state
  std::vector<uint32_t> order_host;
  std::vector<std::pair<uint32_t, uint32_t>> ranges;
  uint32_t bL = 0, brule = 0;
  float balpha = 0.0f;
  DevBuf pair_out, pair_cnt, lids, pair_in;
  DevBuf gtab, gtab_busy;  // second-level visited tables of large-beam searches (search_impl.cuh)
  uint32_t gtab_regions = 0;
  std::mutex gtab_mu;
  PruneHandoff hand;  // the tensor-core prune's hand-off region (this index only)
  std::atomic<uint32_t> max_beam{0};  // search_max_beam, computed once
};

namespace {

void set_device(const gann_index* idx) { cu(cudaSetDevice(idx->device), "cudaSetDevice"); }

gann_index* new_index(uint64_t n, uint32_t d, int elem, int metric, uint32_t R, int device,
                      uint32_t rank = 0, uint32_t nparts = 1) {
  if (elem < GANN_U8 || elem > GANN_F32) fail(GANN_EINVAL, "unknown element kind");
  if (metric != GANN_L2 && metric != GANN_IP) fail(GANN_EINVAL, "unknown metric");
  if (d == 0) fail(GANN_EINVAL, "dimension must be positive");
  if (n > 0 && R == 0) fail(GANN_EINVAL, "graph capacity must be positive");
  if (n >= 0xFFFFFFFFull) fail(GANN_EINVAL, "ids are uint32: n must be below 2^32-1");
  if (R > 1024) fail(GANN_EINVAL, "degree bound above 1024 is not supported");
  auto* idx = new gann_index();
  try {
    idx->device = device;
    idx->n = n;
    idx->d = d;
    idx->elem = elem;
    idx->metric = metric;
    idx->R = R;
    idx->row_bytes = static_cast<uint32_t>(d * elem_bytes(elem));
    idx->stride = (uint64_t(idx->row_bytes) + 15) & ~uint64_t(15);
    if (idx->stride > 2048) fail(GANN_EINVAL, "rows above 2048 bytes are not supported");
    idx->geom = make_geometry(static_cast<uint32_t>(idx->stride / 16));
    if (nparts == 0 || rank >= nparts) fail(GANN_EINVAL, "bad partition rank/count");
    idx->part_rank = rank;
    idx->part_count = nparts;
    idx->part_size = static_cast<uint32_t>((n + nparts - 1) / nparts);
    idx->part_base = static_cast<uint32_t>(std::min<uint64_t>(n, uint64_t(rank) * idx->part_size));
    idx->part_rows = static_cast<uint32_t>(std::min<uint64_t>(n, uint64_t(idx->part_base) + idx->part_size) - idx->part_base);
    set_device(idx);
    cu(cudaStreamCreateWithFlags(&idx->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    const uint64_t nn = std::max<uint64_t>(n, 1);
    const uint64_t rows = std::max<uint64_t>(idx->part_rows, 1);
    cu(cudaMalloc(&idx->points, nn * idx->stride), "cudaMalloc points");
    cu(cudaMalloc(&idx->adj, rows * std::max<uint32_t>(R, 1) * 4), "cudaMalloc graph");
    cu(cudaMalloc(&idx->spre, std::max<uint64_t>(rows, 1)), "cudaMalloc row prefixes");
    cu(cudaMalloc(&idx->tcount, rows * 4), "cudaMalloc tcount");
    cu(cudaMalloc(&idx->tgroup, rows * 4), "cudaMalloc tgroup");
    cu(cudaMalloc(&idx->d_parts, sizeof(uint32_t*) * nparts), "cudaMalloc parts");
    {
      std::vector<uint32_t*> parts(nparts, nullptr);
      parts[rank] = idx->adj;
      cu(cudaMemcpy(idx->d_parts, parts.data(), sizeof(uint32_t*) * nparts, cudaMemcpyHostToDevice), "parts");
    }
    cu(cudaMalloc(&idx->stats, sizeof(unsigned long long) * kStCount * kStatSlots), "cudaMalloc stats");
    cu(cudaMalloc(&idx->counters, sizeof(unsigned long long) * kCntNum), "cudaMalloc counters");
    cu(cudaMalloc(&idx->flags, 16), "cudaMalloc flags");
    cu(cudaMalloc(&idx->qctr, kQueryCounters * 4), "cudaMalloc query counters");
    cu(cudaMemsetAsync(idx->points, 0, nn * idx->stride, idx->stream), "memset");
    cu(cudaMemsetAsync(idx->adj, 0xFF, rows * std::max<uint32_t>(R, 1) * 4, idx->stream), "memset");
    cu(cudaMemsetAsync(idx->spre, 0, std::max<uint64_t>(rows, 1), idx->stream), "memset");
    cu(cudaMemsetAsync(idx->tcount, 0, rows * 4, idx->stream), "memset");
    cu(cudaMemsetAsync(idx->stats, 0, sizeof(unsigned long long) * kStCount * kStatSlots, idx->stream), "memset");
    cu(cudaMemsetAsync(idx->flags, 0, 16, idx->stream), "memset");
    // load the kernels this index will launch now rather than at their first
    // launch inside a timed build (internal.h); once per process and kind
    static std::mutex preload_mu;
    static std::set<std::tuple<int, int, int, int, int>> preloaded;
    {
      std::lock_guard<std::mutex> lk(preload_mu);
      if (preloaded.insert({device, elem, metric, idx->geom.lpr, idx->geom.cpl}).second) {
        preload_search(elem, metric, idx->geom);
        preload_prune(elem, metric, idx->geom);
        preload_backedge(elem, metric, idx->geom);
        preload_misc(elem, metric);
      }
    }
  } catch (...) {
    gann_index_free(idx);
    throw;
  }
  return idx;
}

void flush_timers(gann_index* idx);

// The build's batch scratch and the prune hand-off (the index keeps its
// points, graph and query buffers).
void release_build_scratch(gann_index* idx) {
  for (DevBuf* b : {&idx->order, &idx->vis_ids, &idx->vis_d, &idx->nvis, &idx->gtarget, &idx->gcnt, &idx->goff,
                    &idx->gcursor, &idx->gsrc, &idx->poff, &idx->plen, &idx->pid, &idx->pdist, &idx->bigg,
                    &idx->pls, &idx->plb, &idx->bins})
    b->release();
  prune_release(&idx->hand, idx->stream);
}
// Rows of an imported graph must satisfy set_neighbors (src/graph.cpp:42-59)
// and the reference's invariant of distinct neighbours (check_graph_invariants,
// src/graph.cpp:80-92; the search kernel relies on it), checked on the device.
void validate_graph_rows(gann_index* idx, const uint32_t* d_rows, uint64_t rows, uint32_t R, uint64_t n,
                         uint64_t row0, const std::string& what) {
  if (rows == 0) return;
  idx->misc.ensure(64);
  auto* bad = idx->misc.as<unsigned long long>();
  cu(launch_validate_rows(d_rows, rows, R, n, row0, bad, idx->stream), "validate rows");
  unsigned long long b = 0;
  cu(cudaMemcpyAsync(&b, bad, 8, cudaMemcpyDeviceToHost, idx->stream), "read back");
  cu(cudaStreamSynchronize(idx->stream), "stream sync");
  if (b == ~0ull) return;
  const uint64_t v = row0 + (b >> 3);
  static const char* why[] = {"", "id after GANN_NONE padding", "neighbor id out of range", "self loop",
                              "duplicate neighbor"};
  fail(GANN_EINVAL, what + why[b & 7] + " at vertex " + std::to_string(v));
}

// Stream sync; the phase events recorded before it are complete, so their
// times are collected here at no extra cost.
void sync(gann_index* idx) {
  cu(cudaStreamSynchronize(idx->stream), "stream sync");
  flush_timers(idx);
}

template <class T>
T read_dev(gann_index* idx, const T* p) {
  T v;
  cu(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, idx->stream), "read back");
  sync(idx);
  return v;
}

// Stage nq rows (row_bytes each, host or device) into a padded device buffer.
const uint8_t* stage_rows(gann_index* idx, DevBuf& buf, const void* src, uint32_t nq, bool device) {
  buf.ensure(size_t(nq) * idx->stride);
  if (nq == 0) return buf.as<uint8_t>();
  if (idx->stride != idx->row_bytes)
    cu(cudaMemsetAsync(buf.p, 0, size_t(nq) * idx->stride, idx->stream), "memset staging");
  cu(cudaMemcpy2DAsync(buf.p, idx->stride, src, idx->row_bytes, idx->row_bytes, nq,
                       device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, idx->stream),
     "copy rows");
  return buf.as<uint8_t>();
}

// The largest beam the search kernel holds on chip: a warp keeps its query's
// beam (9 B a slot), candidate lists and visited table in shared memory, and
// a CTA (down to one warp for large beams) may use up to the device's opt-in
// maximum (227 KB on a B200): L up to ~24k.
uint32_t search_max_beam(const gann_index* idx) {
  if (const uint32_t c = idx->max_beam.load()) return c;
  static std::mutex mu;
  static std::map<int, int> optin;
  int mx = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = optin.find(idx->device);
    if (it == optin.end()) {
      if (cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, idx->device) != cudaSuccess) mx = 0;
      optin[idx->device] = mx;
    } else {
      mx = it->second;
    }
  }
  uint32_t lo = 0;
  for (uint32_t L = 32; L <= (1u << 20); L += 32) {
    uint32_t lg = 0, bits = 0, ways = 0;
    hash_config(L, idx->n, &lg, &bits, &ways);
    if (search_smem_min_block(L, idx->R, lg, bits != 0) > static_cast<size_t>(mx)) break;
    lo = L;
  }
  const_cast<gann_index*>(idx)->max_beam.store(lo);
  return lo;
}

void validate_search(const gann_index* idx, uint32_t k_out, uint32_t L, uint32_t k_gate,
                     float eps, int mode) {
  // validate_search_args — src/search.cpp:32-48
  if (L == 0 || k_gate == 0) fail(GANN_EINVAL, "beam and k must be positive");
  if (k_gate > L)
    fail(GANN_EINVAL, "k=" + std::to_string(k_gate) + " exceeds beam=" + std::to_string(L));
  if (!(eps >= 0.0f && eps <= 0.25f)) fail(GANN_EINVAL, "epsilon must lie in [0, 0.25]");
  if (k_out > k_gate) fail(GANN_EINVAL, "k_out must not exceed k (the expansion gate)");
  if (mode != GANN_VISITED_FAST && mode != GANN_VISITED_REF && mode != GANN_VISITED_EXACT)
    fail(GANN_EINVAL, "unknown visited mode");
  if (idx->n > 0 && idx->start >= idx->n) fail(GANN_EINVAL, "start vertex out of range");
  if (idx->n > 0x7FFFFFFFull) fail(GANN_EINVAL, "search holds ids in 31 bits: n must be below 2^31");
  if (L > 32) {
    const uint32_t mx = search_max_beam(idx);
    if (L > mx)
      fail(GANN_EINVAL, "beam " + std::to_string(L) + " exceeds the on-chip beam limit " + std::to_string(mx) +
                            " of this index (gann_search_max_beam)");
  }
}

SearchArgs base_search_args(gann_index* idx, uint32_t L, uint32_t k_gate, uint32_t k_out, float eps,
                            int mode) {
  SearchArgs a{};
  a.data = idx->points;
  a.stride = idx->stride;
  a.n = static_cast<uint32_t>(idx->n);
  a.graph = GraphView{idx->adj, idx->d_parts, idx->part_size, idx->part_count, idx->part_base};
  a.R = idx->R;
  a.start = idx->start;
  a.L = L;
  a.k_gate = k_gate;
  a.k_out = k_out;
  a.eps = eps;
  a.visited_mode = mode;
  hash_config(L, idx->n, &a.hash_log2, &a.hash_bits, &a.hash_ways);
  a.dim = idx->d;
  a.row_bytes = idx->row_bytes;
  a.overflow = idx->flags;
  // each launch pulls queries from its own counter: launches on different
  // streams may run concurrently (up to kQueryCounters in flight)
  a.next_query = idx->qctr + (idx->qslot.fetch_add(1) % kQueryCounters);
  a.stats = idx->stats;
  // Large beams use the second-level visited table instead of the shared one
  // (launch_one drops the shared table then): one 32 KB region per resident
  // warp, twice the device's warp slots so concurrent launches find free
  // regions. Where it pays was measured per beam at c1 (serial launch of
  // 10k queries, shared table only -> second level only, ms): 640: 13.4 ->
  // 12.9, 704: 14.7 -> 13.9, 768: 17.0 -> 14.7, 832: 18.4 -> 15.5, 896: 19.7 ->
  // 21.1, 960: 20.9 -> 22.1, 1024: 22.6 -> 24.2, 1280: 29.4 -> 26.9, 1600: 41.8
  // -> 34.7 (the shared memory it frees is worth a resident CTA at some
  // beams and not at others); 400 / 512: 7.9 / 10.0 with the shared table
  // alone. So from GANN_GTAB_MIN_L (default 576; 0 = never) except 896-1151.
  const uint32_t gmin = env_u32("GANN_GTAB_MIN_L", 576);  // read per call (A/B runs flip it)
  const bool gband = L >= 896 && L < 1152 && !env_u32("GANN_GTAB_NO_BAND", 0);
  const uint32_t glog2 = std::min<uint32_t>(kGtabLog2, std::max<uint32_t>(8, env_u32("GANN_GTAB_LOG2", kGtabLog2Default)));
  a.next_pf = static_cast<int>(env_u32("GANN_SEARCH_NEXTPF", 1));
  // Several expansions per step (search_batch.cuh): the Alg. 1 form in the
  // fast mode, R <= 64, ids within the visited table's remainders.
  // GANN_BATCH_EB = 0 turns it off; GANN_BATCH_MIN_L is the smallest beam it takes.
  const uint32_t beb = std::min<uint32_t>(env_u32("GANN_BATCH_EB", 8), 8);
  const uint32_t bcm = std::min<uint32_t>(256, std::max<uint32_t>(64, env_u32("GANN_BATCH_CM", 64) & ~31u));
  const bool batch = beb && mode == GANN_VISITED_FAST && k_gate == L && idx->R <= 64 && L < 65536 &&
                     L >= env_u32("GANN_BATCH_MIN_L", 320) && search_batch_smem_per_warp(L, bcm) <= 200 * 1024;
  // ids beyond the u16 remainders' reach (n > 2^(log2 + 15): 67M at the default
  // region size): the batch kernel's buckets hold two whole ids instead, in
  // the largest regions (GANN_GTAB_WIDE=1 forces it: tests)
  // beams from 1024 evaluate more ids than the default region remembers: the
  // largest region there (c1, 11 -> 12: L = 1024 -2.8%, 2048 -5%, 4096 -7%, 8192 -12% per launch)
  uint32_t blog2 = glog2;
  if (batch && L >= 1024 && !std::getenv("GANN_GTAB_LOG2")) blog2 = kGtabLog2;
  const bool wide = batch && (idx->n > (uint64_t(1) << (blog2 + 15)) || env_u32("GANN_GTAB_WIDE", 0));
  if (batch) {
    a.batch_eb = beb;
    a.batch_cm = bcm;
    a.batch_policy = static_cast<int>(env_u32("GANN_BATCH_POLICY", 1));
  }
  if (batch || (mode == GANN_VISITED_FAST && gmin && L >= gmin && !gband && idx->n <= (uint64_t(1) << (glog2 + 15)))) {
    std::lock_guard<std::mutex> lk(idx->gtab_mu);
    if (!idx->gtab_regions) {
      int sms = 148, warps = 64;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, idx->device);
      cudaDeviceGetAttribute(&warps, cudaDevAttrMaxThreadsPerMultiProcessor, idx->device);
      const uint32_t regions = 2u * static_cast<uint32_t>(sms) * static_cast<uint32_t>(warps / 32);
      idx->gtab.ensure(size_t(regions) << (kGtabLog2 + 3));
      idx->gtab_busy.ensure(size_t((regions + 31) / 32) * 4);
      cu(cudaMemsetAsync(idx->gtab_busy.p, 0, size_t((regions + 31) / 32) * 4, idx->stream), "memset");
      cu(cudaStreamSynchronize(idx->stream), "sync");
      idx->gtab_regions = regions;
    }
    a.gtab = idx->gtab.as<uint64_t>();
    a.gtab_busy = idx->gtab_busy.as<uint32_t>();
    a.gtab_regions = idx->gtab_regions;
    a.gtab_log2 = wide ? kGtabLog2 : (batch ? blog2 : glog2);
    a.gtab_wide = wide ? 1 : 0;
    a.gtab_keep = static_cast<int>(env_u32("GANN_GTAB_KEEP", 1));

  }
  return a;
}

// Launch the search over nq queries, chunking in REF mode so the L*L tables
// stay under ~1 GiB.
void run_search(gann_index* idx, SearchArgs a, cudaStream_t s) {
  if (a.visited_mode == GANN_VISITED_EXACT) {
    uint32_t ts = 4096;
    while (ts < 512u * a.L) ts <<= 1;
    a.exact_slots = ts;
  }
  if (a.visited_mode == GANN_VISITED_REF || a.visited_mode == GANN_VISITED_EXACT) {
    const uint64_t per = (a.visited_mode == GANN_VISITED_REF ? uint64_t(a.L) * a.L : a.exact_slots) * 4;
    const uint32_t chunk = static_cast<uint32_t>(std::max<uint64_t>(1, (1ull << 30) / per));
    idx->table.ensure(std::min<uint64_t>(chunk, std::max<uint32_t>(a.nq, 1)) * per);
    const uint32_t nq = a.nq;
    for (uint32_t q0 = 0; q0 < nq; q0 += chunk) {
      SearchArgs c = a;
      c.nq = std::min(chunk, nq - q0);
      c.ref_table = idx->table.as<uint32_t>();
      if (c.queries) c.queries += uint64_t(q0) * a.stride;
      if (c.query_rows) c.query_rows += q0;
      if (c.start_override) c.start_override += q0;
      if (c.out_ids) c.out_ids += uint64_t(q0) * a.k_out, c.out_dists += uint64_t(q0) * a.k_out;
      if (c.n_visited) c.n_visited += q0;
      if (c.dist_comps) c.dist_comps += q0;
      if (c.vis_ids) c.vis_ids += uint64_t(q0) * a.vcap, c.vis_dists += uint64_t(q0) * a.vcap;
      cu(launch_search(c, idx->elem, idx->metric, idx->geom, s), "search kernel");
    }
    return;
  }
  cu(launch_search(a, idx->elem, idx->metric, idx->geom, s), "search kernel");
}

// Lists up to kPruneSmallCap are pruned by one warp; longer ones by the
// chunked CTA kernel (any length). Back-edge groups up to kSmallGroupCap
// sources are merged by one warp with an in-order sort; bigger (hub) groups of
// the batch form need no order (they always re-prune). kSortedGroupCap bounds
// the order-preserving path for explicit pairs (group_by_key,
// apply_back_edges with possibly repeated pairs).
constexpr uint32_t kPruneSmallCap = 512;
constexpr uint32_t kSmallGroupCap = 256;
constexpr uint32_t kSortedGroupCap = 32768;

PruneArgs base_prune_args(gann_index* idx, float alpha, int rule) {
  // a row prefix is mutually non-culling only under the (alpha, rule) that
  // pruned it: a launch with other parameters forgets every prefix first
  if (alpha != idx->spre_alpha || rule != idx->spre_rule) {
    cu(cudaMemsetAsync(idx->spre, 0, std::max<uint64_t>(idx->part_rows, 1), idx->stream), "clear row prefixes");
    idx->spre_alpha = alpha;
    idx->spre_rule = rule;
  }
  PruneArgs p{};
  p.data = idx->points;
  p.stride = idx->stride;
  p.R = idx->R;
  p.alpha = alpha;
  p.rule = rule;
  p.too_long = idx->flags + 1;
  p.stats = idx->stats;
  // kernels writing rows into out_adj record the prune prefix (GANN_NO_SPRE=1:
  // no prefixes, every re-prune tests all pairs — an A/B switch for tests)
  static const bool no_spre = env_u32("GANN_NO_SPRE", 0) != 0;
  p.spre = no_spre ? nullptr : idx->spre;
  p.hand = &idx->hand;
  return p;
}

void check_prune_params(float alpha, int rule) {
  if (!(alpha > 0.0f)) fail(GANN_EINVAL, "alpha must be positive");  // prune.cpp:12
  if (rule != GANN_SCALE_CANDIDATE && rule != GANN_SCALE_SELECTED) fail(GANN_EINVAL, "unknown prune rule");
}

// Phase timer of the build: a pair of events on the index's stream. stop()
// does not wait; the elapsed times are added to build_ms[phase] when the
// build ends (flush_timers), so the phases add no host round trips.
struct Timer {
  cudaEvent_t a, b;
  cudaStream_t s;
  explicit Timer(cudaStream_t st) : s(st) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  void stop(gann_index* idx, int phase);  // phase < 0: not accumulated
};

void Timer::stop(gann_index* idx, int phase) {
  cudaEventRecord(b, s);
  idx->timers.emplace_back(a, b, phase);
}

// Waits for the recorded phase events and adds their times to build_ms.
void flush_timers(gann_index* idx) {
  for (auto& [a, b, phase] : idx->timers) {
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (phase >= 0) idx->build_ms[phase] += ms;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  idx->timers.clear();
}

// alpha_prune over lists of length <= maxlen, each by the smallest kernel that
// fits: integer rows on the tensor-core kernel in 128/256/512 bins, f32 rows
// on the warp kernel; anything longer on the chunked kernel.
void prune_binned(gann_index* idx, PruneArgs p, uint32_t maxlen, bool fine = false) {
  if (p.count == 0) return;
  const bool mma = prune_uses_mma(idx->elem, std::min<uint32_t>(maxlen, 512), idx->stride, idx->R) &&
                   !std::getenv("GANN_NO_MMA");
  // bins: (0,128] (128,256] (256,512] on the tensor cores, or (0,512] on the
  // warp kernel for f32; then anything longer on the chunked kernel
  const uint32_t bin0 = env_u32("GANN_PRUNE_BIN0", 80);  // a first, smaller tensor-core bin (0: none)
  // the staging area of a bin is sized by its bound, so finer bins fit more
  // CTAs per SM; insert-time lists (|V| ~ 1.3 L, spread out) take the finer
  // set (-16% prune time at c1 against 128/256/512), re-prune lists (a row
  // plus a few sources) the coarser one (their extra launches cost more)
  std::vector<uint32_t> bounds;
  if (!mma)
    bounds = {kPruneSmallCap};
  else if (fine)
    bounds = {bin0 ? bin0 : 80, 128, 160, 192, 224, 256, 320, 512};
  else
    bounds = {bin0 ? bin0 : 80, 128, 192, 256, 512};
  const int nb = static_cast<int>(bounds.size());
  // back-edge re-prunes of a row prefix plus a few entries: the warp kernel
  // (integer rows, R <= 64; GANN_SMALL_REPRUNE=0 sends them to the bins)
  static const bool small_on = env_u32("GANN_SMALL_REPRUNE", 1) != 0;
  const bool small = mma && p.row_lists && p.spre && idx->R <= 64 && small_on;
  p.small_u = small ? reprune_small_max_u() : 0u;
  // ... in two classes: lists with at most 2 such entries run a smaller instance (GANN_SMALL_U2=0: one class)
  static const bool small2_on = env_u32("GANN_SMALL_U2", 1) != 0;
  p.small_u2 = small && small2_on ? reprune_small_low_u() : 0u;
  idx->bins.ensure(size_t(p.count) * (nb + 2) * 4 + 64 * 4);
  uint32_t* d_counts = idx->bins.as<uint32_t>();
  uint32_t* d_bounds = d_counts + 16;
  uint32_t* d_lists = d_counts + 64;
  cu(cudaMemcpyAsync(d_bounds, bounds.data(), bounds.size() * 4, cudaMemcpyHostToDevice, idx->stream), "bins");
  cu(launch_bin_lists(p, d_bounds, nb, d_counts, d_lists, idx->stream), "bin lists");
  uint32_t counts[16] = {};
  cu(cudaMemcpyAsync(counts, d_counts, (nb + 2) * 4, cudaMemcpyDeviceToHost, idx->stream), "bin counts");
  sync(idx);
  uint32_t lo = 0, total = 0;
  if (p.small_u && std::getenv("GANN_PRUNE_DEBUG")) {
    static unsigned long long acc[3] = {0, 0, 0};
    acc[0] += counts[nb];
    acc[1] += counts[nb + 1];
    acc[2] += p.count;
    std::fprintf(stderr, "re-prune lists so far: %llu with <= 2 extra entries, %llu with 3-4, %llu in all\n", acc[0], acc[1], acc[2]);
  }
  for (int c = nb; c <= nb + 1; c++) {
    if (!counts[c]) continue;
    PruneArgs q = p;
    q.list_index = d_lists + size_t(c) * p.count;
    q.count = counts[c];
    q.small_u = c == nb ? p.small_u2 : p.small_u;  // selects the instance
    cu(launch_reprune_small(q, idx->elem, idx->metric, idx->geom, idx->stream), "re-prune (warp)");
    total += counts[c];
  }
  for (int b = 0; b < nb; b++) {
    total += counts[b];
    if (counts[b]) {
      PruneArgs q = p;
      q.list_index = d_lists + size_t(b) * p.count;
      q.count = counts[b];
      q.mmin = lo + 1;
      q.mcap = std::min(bounds[b], maxlen);
      q.skip_long = 0;
      cu(launch_prune(q, idx->elem, idx->metric, idx->geom, 32, idx->stream),
         mma ? "prune kernel (tensor cores)" : "prune kernel");
    }
    lo = bounds[b];
  }
  if (total < p.count) {  // the rest is longer than the last bound
    // lists longer than maxlen (insert-time walks that outgrew the visited
    // buffer: only maxlen entries were written) are skipped here; the search
    // flagged them and insert_batch re-runs them with a larger buffer
    PruneArgs q = p;
    q.mmin = lo + 1;
    q.mcap = maxlen;
    q.skip_long = 1;
    cu(launch_prune(q, idx->elem, idx->metric, idx->geom, 256, idx->stream), "prune kernel (chunked)");
  }
}

// Insert points order[lo..hi) (device ids) against the current graph:
// search {L, L, 0} + alpha_prune of each visited list into its row.
void insert_batch(gann_index* idx, const uint32_t* d_ids, uint32_t B, uint32_t L, float alpha,
                  int rule, bool timed) {
  if (B == 0) return;
  const uint32_t vcap = std::max<uint32_t>(1, env_u32("GANN_VCAP", std::max<uint32_t>(64, 3 * L)));
  idx->vis_ids.ensure(size_t(B) * vcap * 4);
  idx->vis_d.ensure(size_t(B) * vcap * 4);
  idx->nvis.ensure(size_t(B) * 4);
  cu(cudaMemsetAsync(idx->flags, 0, 8, idx->stream), "memset flags");
  // GANN_BUILD_VISITED=exact: the build's searches count distinct evaluations
  // (a diagnostic for the build roofline's algorithmic bytes; the graph is
  // the same in every visited mode)
  const char* bv = std::getenv("GANN_BUILD_VISITED");
  const int bmode = bv && std::string(bv) == "exact" ? GANN_VISITED_EXACT : GANN_VISITED_FAST;
  SearchArgs a = base_search_args(idx, L, L, 0, 0.0f, bmode);
  a.query_rows = d_ids;
  a.nq = B;
  a.n_visited = idx->nvis.as<uint32_t>();
  a.vis_ids = idx->vis_ids.as<uint32_t>();
  a.vis_dists = idx->vis_d.as<float>();
  a.vcap = vcap;
  Timer ts(idx->stream);
  run_search(idx, a, idx->stream);
  ts.stop(idx, timed ? 1 : -1);
  PruneArgs p = base_prune_args(idx, alpha, rule);
  p.count = B;
  p.points = d_ids;
  p.fixed_stride = vcap;
  p.lengths = idx->nvis.as<uint32_t>();
  p.cand_ids = idx->vis_ids.as<uint32_t>();
  p.cand_dists = idx->vis_d.as<float>();
  p.out_adj = idx->adj;
  p.out_base = idx->part_base;
  p.mcap = vcap;
  Timer tp(idx->stream);
  prune_binned(idx, p, vcap, true);
  tp.stop(idx, timed ? 2 : -1);
  uint32_t fl[2];
  cu(cudaMemcpyAsync(fl, idx->flags, 8, cudaMemcpyDeviceToHost, idx->stream), "read flags");
  sync(idx);
  if (fl[0] == 0) return;
  // Rare long walks (|V| > vcap): their lists were skipped by the prune. Re-run
  // exactly those searches with room for the whole visited list — the graph
  // they read is unchanged (batch points are unreachable until phase 2), so
  // the walk is the same — and prune them with the any-length kernel.
  std::vector<uint32_t> nv(B), ids(B);
  cu(cudaMemcpyAsync(nv.data(), idx->nvis.p, size_t(B) * 4, cudaMemcpyDeviceToHost, idx->stream), "read |V|");
  cu(cudaMemcpyAsync(ids.data(), d_ids, size_t(B) * 4, cudaMemcpyDeviceToHost, idx->stream), "read ids");
  sync(idx);
  std::vector<uint32_t> redo;
  uint32_t vmax = 0;
  for (uint32_t b = 0; b < B; b++)
    if (nv[b] > vcap) {
      redo.push_back(ids[b]);
      vmax = std::max(vmax, nv[b]);
    }
  const uint32_t nr = static_cast<uint32_t>(redo.size());
  const uint32_t vcap2 = vmax;
  idx->pt.ensure(size_t(nr) * 4);
  cu(cudaMemcpyAsync(idx->pt.p, redo.data(), size_t(nr) * 4, cudaMemcpyHostToDevice, idx->stream), "upload");
  idx->vis_ids.ensure(size_t(nr) * vcap2 * 4);
  idx->vis_d.ensure(size_t(nr) * vcap2 * 4);
  cu(cudaMemsetAsync(idx->flags, 0, 8, idx->stream), "memset flags");
  SearchArgs a2 = a;
  a2.query_rows = idx->pt.as<uint32_t>();
  a2.nq = nr;
  a2.vis_ids = idx->vis_ids.as<uint32_t>();
  a2.vis_dists = idx->vis_d.as<float>();
  a2.vcap = vcap2;
  a2.stats = nullptr;  // counted once already
  run_search(idx, a2, idx->stream);
  PruneArgs p2 = p;
  p2.count = nr;
  p2.points = idx->pt.as<uint32_t>();
  p2.fixed_stride = vcap2;
  p2.cand_ids = a2.vis_ids;
  p2.cand_dists = a2.vis_dists;
  prune_binned(idx, p2, vcap2);
  cu(cudaMemcpyAsync(fl, idx->flags, 8, cudaMemcpyDeviceToHost, idx->stream), "read flags");
  sync(idx);
  if (fl[0] || fl[1]) fail(GANN_ECUDA, "long-walk re-run overflowed its visited buffer");
}

// Phase 2: group reverse pairs by target and merge (apply_back_edges).
// Batch form (bsrc != nullptr): the pairs are the out-rows of bsrc[0..B).
void apply_back(gann_index* idx, const uint32_t* bsrc, uint32_t B, const uint32_t* ptarget,
                const uint32_t* psource, uint64_t npairs, float alpha, int rule, bool timed,
                uint32_t* out_keys = nullptr, uint32_t* out_vals = nullptr,
                uint64_t* ngroups_out = nullptr, const uint32_t* key_of_target = nullptr,
                const uint32_t* pordinal = nullptr, uint32_t pstride = 1, bool explicit_distinct = false) {
  if (npairs == 0) {
    if (ngroups_out) *ngroups_out = 0;
    return;
  }
  if (npairs >= 0xFFFFFFFFull) fail(GANN_EINVAL, "too many reverse pairs in one batch");
  const uint32_t R = idx->R;
  BackEdgeArgs b{};
  b.data = idx->points;
  b.stride = idx->stride;
  b.adj = idx->adj;
  b.base = idx->part_base;
  b.pstride = pstride;
  b.pordinal = pordinal;
  b.R = R;
  b.bsrc = bsrc;
  b.B = B;
  b.ptarget = ptarget;
  b.psource = psource;
  b.npairs = npairs;
  b.sources_distinct = bsrc != nullptr || explicit_distinct;
  b.tcount = idx->tcount;
  b.tgroup = idx->tgroup;
  b.counters = idx->counters;
  // groups above small_group_cap sources take the hub merge, which assumes
  // the merged list overflows R: so the cap is at least R (R up to 1024)
  b.small_group_cap = std::max<uint32_t>(kSmallGroupCap, idx->R);
  b.big_group_cap = kSortedGroupCap;
  b.prune_small_cap = kPruneSmallCap;
  b.small_dists = !prune_uses_mma(idx->elem, kPruneSmallCap, idx->stride, R) || std::getenv("GANN_NO_MMA");
  b.key_of_target = key_of_target;
  cu(cudaMemsetAsync(idx->counters, 0, sizeof(unsigned long long) * kCntNum, idx->stream), "memset");
  const uint64_t gmax = npairs;  // groups <= pairs
  idx->gtarget.ensure(gmax * 4);
  b.gtarget = idx->gtarget.as<uint32_t>();
  Timer tg(idx->stream);
  cu(backedge_count(b, idx->stream), "back-edge count");
  const uint32_t ng = static_cast<uint32_t>(read_dev(idx, idx->counters + kCntGroups));
  idx->gcnt.ensure(size_t(ng) * 4);
  idx->goff.ensure(size_t(ng) * 8);
  idx->gcursor.ensure(size_t(ng) * 4);
  idx->gsrc.ensure(npairs * 4);
  idx->poff.ensure(size_t(ng) * 8);
  idx->plen.ensure(size_t(ng) * 4);
  idx->bigg.ensure(size_t(ng) * 4);
  idx->pls.ensure(size_t(ng) * 4);
  idx->plb.ensure(size_t(ng) * 4);
  const uint64_t ptotal = uint64_t(ng) * R + npairs;
  idx->pid.ensure(ptotal * 4);
  idx->pdist.ensure(ptotal * 4);
  b.gcnt = idx->gcnt.as<uint32_t>();
  b.goff = idx->goff.as<uint64_t>();
  b.gcursor = idx->gcursor.as<uint32_t>();
  b.gsrc = idx->gsrc.as<uint32_t>();
  b.poff = idx->poff.as<uint64_t>();
  b.plen = idx->plen.as<uint32_t>();
  b.pid = idx->pid.as<uint32_t>();
  b.pdist = idx->pdist.as<float>();
  b.big_groups = idx->bigg.as<uint32_t>();
  b.plist_small = idx->pls.as<uint32_t>();
  b.plist_big = idx->plb.as<uint32_t>();
  cu(backedge_offsets(b, ng, idx->stream), "back-edge offsets");
  cu(backedge_scatter(b, idx->stream), "back-edge scatter");
  unsigned long long cnt[kCntNum];
  cu(cudaMemcpyAsync(cnt, idx->counters, sizeof(cnt), cudaMemcpyDeviceToHost, idx->stream), "read");
  sync(idx);
  const uint32_t nbig = static_cast<uint32_t>(cnt[kCntBig]);
  if ((out_keys || !b.sources_distinct) && cnt[kCntMaxGroup] > kSortedGroupCap)
    fail(GANN_EINVAL, "a group of " + std::to_string(cnt[kCntMaxGroup]) + " pairs exceeds the ordered-group cap " +
                          std::to_string(kSortedGroupCap));
  tg.stop(idx, timed ? 3 : -1);
  if (out_keys) {  // group_by_key mode
    cu(backedge_write_groups(b, ng, nbig, out_keys, out_vals, idx->stream), "group write");
    sync(idx);
    if (ngroups_out) *ngroups_out = ng;
    return;
  }
  Timer tm(idx->stream);
  cu(backedge_merge(b, ng, nbig, idx->elem, idx->metric, idx->geom, idx->stream), "back-edge merge");
  cu(cudaMemcpyAsync(cnt, idx->counters, sizeof(cnt), cudaMemcpyDeviceToHost, idx->stream), "read");
  sync(idx);
  tm.stop(idx, timed ? 4 : -1);
  if (cnt[kCntTooBig]) fail(GANN_ECUDA, "back-edge group exceeded the merge capacity");
  const uint32_t nps = static_cast<uint32_t>(cnt[kCntPruneSmall]);
  const uint32_t npb = static_cast<uint32_t>(cnt[kCntPruneBig]);
  idx->back_pairs += npairs;
  idx->back_groups += ng;
  idx->back_pruned += nps + npb;
  Timer tp(idx->stream);
  PruneArgs p = base_prune_args(idx, alpha, rule);
  p.points = b.gtarget;
  p.begins = b.poff;
  p.lengths = b.plen;
  p.cand_ids = b.pid;
  p.cand_dists = b.pdist;
  p.out_adj = idx->adj;
  p.out_base = idx->part_base;
  p.row_lists = 1;  // merged lists start with the target's current row
  cu(cudaMemsetAsync(idx->flags + 1, 0, 4, idx->stream), "memset flags");
  if (nps) {
    p.count = nps;
    p.list_index = b.plist_small;
    p.cand_dists = b.small_dists ? b.pdist : nullptr;  // nullptr: the prune computes d(t, .)
    prune_binned(idx, p, kPruneSmallCap);
    p.cand_dists = b.pdist;
  }
  if (npb) {
    p.count = npb;
    p.list_index = b.plist_big;
    p.mmin = 0;
    p.mcap = 0xFFFFFFFFu;
    cu(launch_prune(p, idx->elem, idx->metric, idx->geom, 256, idx->stream), "reprune big");
  }
  uint32_t tl = 0;  // a re-prune list the kernels could not take (must not happen)
  cu(cudaMemcpyAsync(&tl, idx->flags + 1, 4, cudaMemcpyDeviceToHost, idx->stream), "read flags");
  sync(idx);
  if (tl) fail(GANN_ECUDA, "re-prune: " + std::to_string(tl) + " list(s) not taken by any prune kernel");
  tp.stop(idx, timed ? 5 : -1);
}

std::vector<std::pair<uint32_t, uint32_t>> batch_ranges(uint64_t n, uint32_t cap) {
  // src/builder_common.cpp:13-20, + the optional cap hi = min(2 lo, lo + cap, n)
  std::vector<std::pair<uint32_t, uint32_t>> r;
  for (uint64_t lo = 1; lo < n;) {
    uint64_t hi = std::min<uint64_t>(lo << 1, n);
    if (cap) hi = std::min<uint64_t>(hi, lo + cap);
    r.emplace_back(static_cast<uint32_t>(lo), static_cast<uint32_t>(hi));
    lo = hi;
  }
  return r;
}

uint32_t choose_start_dev(gann_index* idx) {
  if (idx->n == 0) fail(GANN_EINVAL, "cannot pick a start point of an empty dataset");
  idx->misc.ensure(sizeof(double) * idx->d + sizeof(float) * idx->d + 16);
  double* colsum = idx->misc.as<double>();
  float* centroid = reinterpret_cast<float*>(colsum + idx->d);
  unsigned long long* best = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(centroid + idx->d) + 15) & ~uintptr_t(15));
  idx->misc.ensure(reinterpret_cast<uint8_t*>(best + 1) - idx->misc.as<uint8_t>());
  colsum = idx->misc.as<double>();
  centroid = reinterpret_cast<float*>(colsum + idx->d);
  best = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(centroid + idx->d) + 15) & ~uintptr_t(15));
  cu(launch_choose_start(idx->points, idx->stride, idx->n, idx->d, idx->elem, idx->metric, colsum,
                         centroid, best, idx->stream),
     "choose_start");
  const unsigned long long k = read_dev(idx, best);
  return static_cast<uint32_t>(k & 0xFFFFFFFFu);
}

// Brute force over padded query rows — compute_groundtruth (src/dataset.cpp:172-217).
void run_groundtruth(gann_index* idx, const uint8_t* q, uint32_t nq, uint32_t k, uint32_t* d_ids,
                     float* d_dists, cudaStream_t s) {
  if (k == 0 || k > 64) fail(GANN_EINVAL, "groundtruth: k must lie in [1, 64]");
  if (k > idx->n) fail(GANN_EINVAL, "groundtruth: k=" + std::to_string(k) + " exceeds n");
  if (idx->stride > 1568) fail(GANN_EINVAL, "groundtruth: rows above 1568 bytes are not supported");
  if (nq == 0) return;
  const uint32_t splits = groundtruth_splits(idx->n, nq);
  idx->gt.ensure(size_t(nq) * splits * (k <= 16 ? 16 : 64) * 8);
  cu(launch_groundtruth(idx->points, idx->stride, idx->n, q, nq, k, idx->elem, idx->metric,
                        static_cast<uint32_t>(idx->stride / 16), idx->gt.as<unsigned long long>(),
                        splits, d_ids, d_dists, s),
     "groundtruth kernel");
}

}  // namespace

extern "C" {

const char* gann_last_error(void) { return g_err.c_str(); }
const char* gann_version(void) { return "gann 0.1 sm_100a"; }

int gann_index_create(const void* points, uint64_t n, uint32_t d, int elem, int metric, uint32_t R,
                      int device, gann_index** out) {
  return guarded([&] {
    if (!out) fail(GANN_EINVAL, "out is NULL");
    if (n && !points) fail(GANN_EINVAL, "points is NULL");
    gann_index* idx = new_index(n, d, elem, metric, R, device);
    try {
      if (n) {
        cu(cudaMemcpy2DAsync(idx->points, idx->stride, points, idx->row_bytes, idx->row_bytes, n,
                             cudaMemcpyHostToDevice, idx->stream),
           "upload points");
      }
      sync(idx);
    } catch (...) {
      gann_index_free(idx);
      throw;
    }
    *out = idx;
  });
}

int gann_index_create_device(const void* d_points, uint64_t n, uint32_t d, int elem, int metric,
                             uint32_t R, int device, gann_index** out) {
  return guarded([&] {
    if (!out) fail(GANN_EINVAL, "out is NULL");
    gann_index* idx = new_index(n, d, elem, metric, R, device);
    try {
      if (n) {
        cu(cudaMemcpy2DAsync(idx->points, idx->stride, d_points, idx->row_bytes, idx->row_bytes, n,
                             cudaMemcpyDeviceToDevice, idx->stream),
           "copy points");
      }
      sync(idx);
    } catch (...) {
      gann_index_free(idx);
      throw;
    }
    *out = idx;
  });
}

void gann_index_free(gann_index* idx) {
  if (!idx) return;
  cudaSetDevice(idx->device);
  if (idx->stream) cudaStreamSynchronize(idx->stream);
  flush_timers(idx);
  for (void* p : idx->ipc_open)
    if (p) cudaIpcCloseMemHandle(p);
  if (idx->d_parts) cudaFree(idx->d_parts);
  for (DevBuf* b : {&idx->pair_out, &idx->pair_cnt, &idx->lids, &idx->pair_in, &idx->gtab, &idx->gtab_busy})
    b->release();
  for (void* p : {static_cast<void*>(idx->points), static_cast<void*>(idx->adj),
                  static_cast<void*>(idx->tcount), static_cast<void*>(idx->tgroup),
                  static_cast<void*>(idx->stats), static_cast<void*>(idx->counters),
                  static_cast<void*>(idx->flags), static_cast<void*>(idx->qctr), static_cast<void*>(idx->spre)})
    if (p) cudaFree(p);
  for (DevBuf* b : {&idx->q, &idx->qstaged, &idx->qids, &idx->qdists, &idx->qnvis, &idx->qdc, &idx->qvids,
                    &idx->qvd, &idx->qstart, &idx->table, &idx->order, &idx->vis_ids, &idx->vis_d,
                    &idx->nvis, &idx->gtarget, &idx->gcnt, &idx->goff, &idx->gcursor, &idx->gsrc,
                    &idx->poff, &idx->plen, &idx->pid, &idx->pdist, &idx->bigg, &idx->pls,
                    &idx->plb, &idx->pt, &idx->ps, &idx->ok, &idx->ov, &idx->misc, &idx->gt, &idx->bins})
    b->release();
  prune_release(&idx->hand, idx->stream);
  if (idx->stream) cudaStreamDestroy(idx->stream);
  delete idx;
}

int gann_index_info(const gann_index* idx, uint64_t* n, uint32_t* d, int* elem, int* metric,
                    uint32_t* R, uint32_t* start) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    if (n) *n = idx->n;
    if (d) *d = idx->d;
    if (elem) *elem = idx->elem;
    if (metric) *metric = idx->metric;
    if (R) *R = idx->R;
    if (start) *start = idx->start;
  });
}

int gann_build(gann_index* idx, uint32_t L, float alpha, int rule, uint64_t seed, uint32_t max_batch) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    // src/diskann.cpp:33-42
    if (idx->n == 0) fail(GANN_EINVAL, "cannot build over an empty dataset");
    if (L == 0 || idx->R == 0) fail(GANN_EINVAL, "build beam and degree bound must be positive");
    if (idx->n > 0x7FFFFFFFull) fail(GANN_EINVAL, "search holds ids in 31 bits: n must be below 2^31");
    if (L > 32 && L > search_max_beam(idx))
      fail(GANN_EINVAL, "build beam " + std::to_string(L) + " exceeds the on-chip beam limit " +
                            std::to_string(search_max_beam(idx)));
    check_prune_params(alpha, rule);
    if (L < idx->R)
      std::fprintf(stderr, "warning: build beam %u below degree bound %u; lists will be thin\n", L,
                   idx->R);
    set_device(idx);
    if (idx->part_count != 1) fail(GANN_EINVAL, "a partitioned index builds with gann_part_build_begin/phase1/phase2");
    for (double& m : idx->build_ms) m = 0;
    idx->back_pairs = idx->back_groups = idx->back_pruned = 0;
    const uint64_t n = idx->n;
    cu(cudaMemsetAsync(idx->adj, 0xFF, n * idx->R * 4, idx->stream), "clear graph");
    cu(cudaMemsetAsync(idx->spre, 0, n, idx->stream), "clear row prefixes");
    cu(cudaMemsetAsync(idx->tcount, 0, n * 4, idx->stream), "clear counts");
    Timer t0(idx->stream);
    // shuffled_order — src/builder_common.cpp:99-107 (same libstdc++ calls):
    // the shuffle does not depend on the start vertex (only the final swap
    // does), so it runs on a host thread while the device picks the start
    // and the batch scratch is allocated
    // (GANN_HOST_SHUFFLE=1: std::shuffle over the array itself, as round 1 did)
    const bool host_shuffle = env_u32("GANN_HOST_SHUFFLE", 0) != 0;
    std::vector<uint32_t> order(n);  // the host shuffle's array, or the swap log
    std::thread shuffler([&] {
      if (!host_shuffle) return shuffle_swap_log(n, mix64(seed, 0x696e73657274ULL), order.data());
      for (uint64_t i = 0; i < n; i++) order[i] = static_cast<uint32_t>(i);
      std::mt19937_64 rng(mix64(seed, 0x696e73657274ULL));
      std::shuffle(order.begin(), order.end(), rng);
    });
    const bool trace_start = env_u32("GANN_TRACE_START", 0) != 0;  // host times of the start phase's steps
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto since = [&](std::chrono::steady_clock::time_point a) {
      return std::chrono::duration<double, std::milli>(now() - a).count();
    };
    const auto ts0 = now();
    uint32_t start = 0;
    try {
      start = choose_start_dev(idx);
    } catch (...) {
      shuffler.join();
      throw;
    }
    idx->start = start;
    const double t_start_vertex = since(ts0);
    const auto ts1 = now();
    // size the per-batch scratch once, from the largest batch: a cudaFree /
    // cudaMalloc inside the loop stalls the device for tens of milliseconds
    try {
      uint32_t bmax = 0;
      for (auto [lo, hi] : batch_ranges(n, max_batch)) bmax = std::max(bmax, hi - lo);
      const uint32_t vcap = std::max<uint32_t>(64, 3 * L);
      const uint64_t pairs = uint64_t(bmax) * idx->R;
      // distinct targets of the largest batch's reverse pairs: at most min(pairs,
      // n), but sizing for that worst case is mostly wasted allocation time (c1:
      // 2.3-2.6M groups per 200k-point batch against a bound of 10M; 5.2 GB of
      // merged-list scratch instead of 2.3 GB, ~100 ms of cudaMalloc in a cold
      // build). A third of the pairs, grown on demand by apply_back / the prune
      // launches if a batch does need more.
      const uint64_t groups = std::min<uint64_t>(std::min<uint64_t>(pairs, n), std::max<uint64_t>(pairs / 3, bmax));
      idx->vis_ids.ensure(size_t(bmax) * vcap * 4);
      idx->vis_d.ensure(size_t(bmax) * vcap * 4);
      idx->nvis.ensure(size_t(bmax) * 4);
      idx->gtarget.ensure(pairs * 4);
      idx->gsrc.ensure(pairs * 4);
      for (DevBuf* b : {&idx->gcnt, &idx->gcursor, &idx->plen, &idx->bigg, &idx->pls, &idx->plb})
        b->ensure(groups * 4);
      idx->goff.ensure(groups * 8);
      idx->poff.ensure(groups * 8);
      const uint64_t ptotal = groups * idx->R + pairs;
      idx->pid.ensure(ptotal * 4);
      idx->pdist.ensure(ptotal * 4);
      if (prune_uses_mma(idx->elem, 512, idx->stride, idx->R))
        prune_reserve(&idx->hand, static_cast<uint32_t>(std::min<uint64_t>(groups, 0xFFFFFFFFu)), idx->stride, idx->R, idx->stream);
      // the prune's length bins: lists x (bins + 1) ids, for the largest count
      // a batch can prune (every group) — growing it batch by batch meant a
      // cudaFree/cudaMalloc pair inside the timed batches
      idx->bins.ensure(size_t(std::max<uint64_t>(groups, bmax)) * 9 * 4 + 64 + 16 * 4);
      idx->order.ensure(n * 4);
    } catch (...) {
      shuffler.join();
      throw;
    }
    const double t_alloc = since(ts1);
    const auto ts2 = now();
    shuffler.join();
    const double t_join = since(ts2);
    const auto ts3 = now();
    if (host_shuffle) {
      std::iter_swap(order.begin(), std::find(order.begin(), order.end(), start));
      cu(cudaMemcpyAsync(idx->order.p, order.data(), n * 4, cudaMemcpyHostToDevice, idx->stream),
         "upload order");
    } else {
      // the permutation from the swap log, on the device (5 n u32 of scratch, freed again)
      DevBuf work;
      work.ensure(n * 5 * 4);
      uint32_t* d_log = work.as<uint32_t>();
      cu(cudaMemcpyAsync(d_log, order.data(), n * 4, cudaMemcpyHostToDevice, idx->stream), "upload swap log");
      void* tmp = nullptr;
      size_t tmp_bytes = 0;
      const cudaError_t e = launch_shuffle_from_log(d_log, n, start, d_log + n, idx->order.as<uint32_t>(), &tmp,
                                                    &tmp_bytes, idx->stream);
      if (e == cudaSuccess) cudaStreamSynchronize(idx->stream);
      if (tmp) cudaFree(tmp);
      work.release();
      cu(e, "shuffle from log");
    }
    t0.stop(idx, 0);
    if (trace_start)
      std::fprintf(stderr, "build start phase (host ms): start vertex %.1f, scratch allocation %.1f, wait for the swap log %.1f, order on the device %.1f\n",
                   t_start_vertex, t_alloc, t_join, since(ts3));
    const uint32_t* d_order = idx->order.as<uint32_t>();
    const bool trace = env_u32("GANN_TRACE", 0) != 0;
    for (auto [lo, hi] : batch_ranges(n, max_batch)) {
      const uint32_t B = hi - lo;
      double before[6];
      std::copy(idx->build_ms, idx->build_ms + 6, before);
      auto t0 = std::chrono::steady_clock::now();
      insert_batch(idx, d_order + lo, B, L, alpha, rule, true);
      apply_back(idx, d_order + lo, B, nullptr, nullptr, uint64_t(B) * idx->R, alpha, rule, true);
      if (trace) {
        const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        std::fprintf(stderr, "batch [%u,%u) wall %.2f ms: search %.2f prune %.2f group %.2f merge %.2f reprune %.2f\n",
                     lo, hi, wall, idx->build_ms[1] - before[1], idx->build_ms[2] - before[2],
                     idx->build_ms[3] - before[3], idx->build_ms[4] - before[4], idx->build_ms[5] - before[5]);
      }
    }
    sync(idx);
    // the batch scratch is sized for the largest batch (tens of GB at 100M
    // points): kept for the next build unless device memory is tight (freeing
    // ~10 GB costs ~0.15 s); gann_release_scratch hands it back on request
    size_t fr = 0, tot = 0;
    cu(cudaMemGetInfo(&fr, &tot), "cudaMemGetInfo");
    if (env_u32("GANN_KEEP_BUILD_SCRATCH", 0) == 0 && fr < tot / 4) release_build_scratch(idx);
  });
}

int gann_release_scratch(gann_index* idx) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    set_device(idx);
    sync(idx);
    release_build_scratch(idx);
  });
}

int gann_build_diskann(const void* points, uint64_t n, uint32_t d, int elem, int metric, uint32_t R,
                       uint32_t L, float alpha, int rule, uint64_t seed, uint32_t max_batch,
                       int device, gann_index** out) {
  gann_index* idx = nullptr;
  int rc = gann_index_create(points, n, d, elem, metric, R, device, &idx);
  if (rc != GANN_OK) return rc;
  rc = gann_build(idx, L, alpha, rule, seed, max_batch);
  if (rc != GANN_OK) {
    gann_index_free(idx);
    return rc;
  }
  *out = idx;
  return GANN_OK;
}

int gann_import_graph(gann_index* idx, const uint32_t* adj, uint32_t start) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    if (idx->part_count != 1) fail(GANN_EINVAL, "import_graph needs an unpartitioned index");
    const uint64_t n = idx->n;
    const uint32_t R = idx->R;
    if (n && start >= n) fail(GANN_EINVAL, "start vertex out of range");
    set_device(idx);
    if (n) cu(cudaMemcpyAsync(idx->adj, adj, n * R * 4, cudaMemcpyHostToDevice, idx->stream), "upload graph");
    try {
      validate_graph_rows(idx, idx->adj, n, R, n, 0, "");
    } catch (...) {  // leave an empty graph, not a half-valid one
      cudaMemsetAsync(idx->adj, 0xFF, n * R * 4, idx->stream);
      cudaStreamSynchronize(idx->stream);
      throw;
    }
    if (n) cu(cudaMemsetAsync(idx->spre, 0, n, idx->stream), "clear row prefixes");  // rows of unknown origin
    idx->start = start;
    sync(idx);
  });
}

int gann_import_graph_device(gann_index* idx, const uint32_t* d_adj, uint32_t start) {
  return guarded([&] {
    if (!idx || (idx->n && !d_adj)) fail(GANN_EINVAL, "NULL argument");
    if (idx->part_count != 1) fail(GANN_EINVAL, "import_graph needs an unpartitioned index");
    if (idx->n && start >= idx->n) fail(GANN_EINVAL, "start vertex out of range");
    set_device(idx);
    validate_graph_rows(idx, d_adj, idx->n, idx->R, idx->n, 0, "");
    if (idx->n)
      cu(cudaMemcpyAsync(idx->adj, d_adj, idx->n * idx->R * 4, cudaMemcpyDeviceToDevice, idx->stream), "copy graph");
    if (idx->n) cu(cudaMemsetAsync(idx->spre, 0, idx->n, idx->stream), "clear row prefixes");
    idx->start = start;
    sync(idx);
  });
}

int gann_export_graph(const gann_index* cidx, uint32_t* adj, uint32_t* deg, uint32_t* start) {
  return guarded([&] {
    gann_index* idx = const_cast<gann_index*>(cidx);
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    set_device(idx);
    const uint64_t n = idx->part_rows;  // a partition exports its own rows
    const uint32_t R = idx->R;
    if (adj && n) {
      cu(cudaMemcpyAsync(adj, idx->adj, n * R * 4, cudaMemcpyDeviceToHost, idx->stream), "download graph");
      sync(idx);
      if (deg)
        for (uint64_t v = 0; v < n; v++) {
          uint32_t k = 0;
          while (k < R && adj[v * R + k] != GANN_NONE) k++;
          deg[v] = k;
        }
    } else if (deg && n) {
      std::vector<uint32_t> tmp(n * R);
      cu(cudaMemcpyAsync(tmp.data(), idx->adj, n * R * 4, cudaMemcpyDeviceToHost, idx->stream), "download graph");
      sync(idx);
      for (uint64_t v = 0; v < n; v++) {
        uint32_t k = 0;
        while (k < R && tmp[v * R + k] != GANN_NONE) k++;
        deg[v] = k;
      }
    }
    if (start) *start = idx->start;
  });
}

int gann_search(gann_index* idx, const void* queries, uint32_t nq, uint32_t k_out, uint32_t L,
                uint32_t k_gate, float eps, int visited_mode, const uint32_t* start_override,
                uint32_t* ids, float* dists, uint32_t* n_visited, uint64_t* dist_comps,
                uint32_t* vis_ids, float* vis_dists, uint32_t vcap) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    validate_search(idx, k_out, L, k_gate, eps, visited_mode);
    if (nq == 0) return;
    if (!queries) fail(GANN_EINVAL, "queries is NULL");
    set_device(idx);
    if (idx->n == 0) {  // src/search.cpp:67 — empty graph, empty result
      for (uint64_t i = 0; i < uint64_t(nq) * k_out; i++) {
        if (ids) ids[i] = GANN_NONE;
        if (dists) dists[i] = __builtin_inff();
      }
      for (uint32_t i = 0; i < nq; i++) {
        if (n_visited) n_visited[i] = 0;
        if (dist_comps) dist_comps[i] = 0;
      }
      return;
    }
    if (start_override)
      for (uint32_t i = 0; i < nq; i++)
        if (start_override[i] >= idx->n) fail(GANN_EINVAL, "start vertex out of range");
    SearchArgs a = base_search_args(idx, L, k_gate, k_out, eps, visited_mode);
    a.queries = stage_rows(idx, idx->q, queries, nq, false);
    a.nq = nq;
    if (start_override) {
      idx->qstart.ensure(size_t(nq) * 4);
      cu(cudaMemcpyAsync(idx->qstart.p, start_override, size_t(nq) * 4, cudaMemcpyHostToDevice, idx->stream), "upload starts");
      a.start_override = idx->qstart.as<uint32_t>();
    }
    if (k_out) {
      idx->qids.ensure(size_t(nq) * k_out * 4);
      idx->qdists.ensure(size_t(nq) * k_out * 4);
      a.out_ids = idx->qids.as<uint32_t>();
      a.out_dists = idx->qdists.as<float>();
    }
    idx->qnvis.ensure(size_t(nq) * 4);
    idx->qdc.ensure(size_t(nq) * 8);
    a.n_visited = idx->qnvis.as<uint32_t>();
    a.dist_comps = idx->qdc.as<uint64_t>();
    if (vis_ids && vcap) {
      idx->qvids.ensure(size_t(nq) * vcap * 4);
      idx->qvd.ensure(size_t(nq) * vcap * 4);
      cu(cudaMemsetAsync(idx->qvids.p, 0xFF, size_t(nq) * vcap * 4, idx->stream), "memset");
      a.vis_ids = idx->qvids.as<uint32_t>();
      a.vis_dists = idx->qvd.as<float>();
      a.vcap = vcap;
    }
    run_search(idx, a, idx->stream);
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
      if (dst) cu(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, idx->stream), "download results");
    };
    if (k_out) {
      d2h(ids, a.out_ids, size_t(nq) * k_out * 4);
      d2h(dists, a.out_dists, size_t(nq) * k_out * 4);
    }
    d2h(n_visited, a.n_visited, size_t(nq) * 4);
    d2h(dist_comps, a.dist_comps, size_t(nq) * 8);
    if (a.vis_ids) {
      d2h(vis_ids, a.vis_ids, size_t(nq) * vcap * 4);
      d2h(vis_dists, a.vis_dists, size_t(nq) * vcap * 4);
    }
    uint32_t no_region = 0;  // search_batch_kernel: warps that found no visited-table region
    d2h(&no_region, idx->flags + 2, 4);
    sync(idx);
    if (no_region) {
      cu(cudaMemsetAsync(idx->flags + 2, 0, 4, idx->stream), "memset flags");
      fail(GANN_ECUDA, "search: no free visited-table region for " + std::to_string(no_region) + " warps");
    }
  });
}

int gann_search_device(gann_index* idx, const void* d_queries, uint32_t nq, uint32_t k_out,
                       uint32_t L, uint32_t k_gate, float eps, int visited_mode, uint32_t* d_ids,
                       float* d_dists, uint32_t* d_n_visited, uint64_t* d_dist_comps, void* stream) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    validate_search(idx, k_out, L, k_gate, eps, visited_mode);
    if (nq == 0) return;
    if (idx->n == 0) fail(GANN_EINVAL, "search over an empty index");
    set_device(idx);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : idx->stream;
    SearchArgs a = base_search_args(idx, L, k_gate, k_out, eps, visited_mode);
    if (idx->stride == idx->row_bytes) {
      a.queries = static_cast<const uint8_t*>(d_queries);
    } else {
      idx->q.ensure(size_t(nq) * idx->stride);
      cu(cudaMemsetAsync(idx->q.p, 0, size_t(nq) * idx->stride, s), "memset");
      cu(cudaMemcpy2DAsync(idx->q.p, idx->stride, d_queries, idx->row_bytes, idx->row_bytes, nq,
                           cudaMemcpyDeviceToDevice, s), "stage queries");
      a.queries = idx->q.as<uint8_t>();
    }
    a.nq = nq;
    a.out_ids = k_out ? d_ids : nullptr;
    a.out_dists = k_out ? d_dists : nullptr;
    a.n_visited = d_n_visited;
    a.dist_comps = d_dist_comps;
    run_search(idx, a, s);
  });
}

int gann_debug_check(int device, uint32_t* failed_line, int* checked_build) {
  return guarded([&] {
    cu(cudaSetDevice(device), "cudaSetDevice");
    cu(cudaDeviceSynchronize(), "sync");
    unsigned v = 0;
    for (unsigned (*f)() : {check_line_search_u8, check_line_search_i8, check_line_search_f32, check_line_prune,
                            check_line_backedge, check_line_misc})
      v = std::max(v, f());
    if (failed_line) *failed_line = v;
#ifdef GANN_CHECKED
    if (checked_build) *checked_build = 1;
#else
    if (checked_build) *checked_build = 0;
#endif
  });
}

int gann_search_max_beam(const gann_index* idx, uint32_t* max_L) {
  return guarded([&] {
    if (!idx || !max_L) fail(GANN_EINVAL, "NULL argument");
    set_device(idx);
    *max_L = search_max_beam(idx);
  });
}

int gann_stage_queries(gann_index* idx, const void* d_queries, uint32_t nq) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    set_device(idx);
    stage_rows(idx, idx->qstaged, d_queries, nq, true);
    idx->staged_nq = nq;
    idx->staged = true;
    sync(idx);
  });
}

int gann_search_staged(gann_index* idx, uint32_t k_out, uint32_t L, uint32_t k_gate, float eps,
                       uint32_t* d_ids, float* d_dists, void* stream) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    validate_search(idx, k_out, L, k_gate, eps, GANN_VISITED_FAST);
    if (idx->n == 0) fail(GANN_EINVAL, "search over an empty index");
    if (!idx->staged) fail(GANN_EINVAL, "no queries staged (call gann_stage_queries first)");
    set_device(idx);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : idx->stream;
    SearchArgs a = base_search_args(idx, L, k_gate, k_out, eps, GANN_VISITED_FAST);
    a.queries = idx->qstaged.as<uint8_t>();
    a.nq = idx->staged_nq;
    a.out_ids = d_ids;
    a.out_dists = d_dists;
    cu(launch_search(a, idx->elem, idx->metric, idx->geom, s), "search kernel");
  });
}

uint64_t gann_search_async_scratch(const gann_index* idx, uint32_t nq, uint32_t k_out) {
  if (!idx) return 0;
  // [counter 256 B][queries nq*stride][ids nq*k_out*4][dists nq*k_out*4]
  return 256 + uint64_t(nq) * idx->stride + uint64_t(nq) * k_out * 8;
}

int gann_search_async(gann_index* idx, const void* h_queries, uint32_t nq, uint32_t k_out, uint32_t L,
                      uint32_t k_gate, float eps, uint32_t* h_ids, float* h_dists, void* d_scratch,
                      uint64_t scratch_bytes, void* stream) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    validate_search(idx, k_out, L, k_gate, eps, GANN_VISITED_FAST);
    if (nq == 0) return;
    if (idx->n == 0) fail(GANN_EINVAL, "search over an empty index");
    if (!h_queries || !d_scratch || (k_out && (!h_ids || !h_dists))) fail(GANN_EINVAL, "NULL argument");
    if (scratch_bytes < gann_search_async_scratch(idx, nq, k_out)) fail(GANN_EINVAL, "scratch too small");
    set_device(idx);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : idx->stream;
    uint8_t* base = static_cast<uint8_t*>(d_scratch);
    uint8_t* dq = base + 256;
    uint32_t* dids = reinterpret_cast<uint32_t*>(dq + uint64_t(nq) * idx->stride);
    float* dd = reinterpret_cast<float*>(dids + uint64_t(nq) * k_out);
    if (idx->stride == idx->row_bytes) {
      cu(cudaMemcpyAsync(dq, h_queries, uint64_t(nq) * idx->stride, cudaMemcpyHostToDevice, s), "upload queries");
    } else {
      cu(cudaMemsetAsync(dq, 0, uint64_t(nq) * idx->stride, s), "memset");
      cu(cudaMemcpy2DAsync(dq, idx->stride, h_queries, idx->row_bytes, idx->row_bytes, nq, cudaMemcpyHostToDevice, s),
         "upload queries");
    }
    SearchArgs a = base_search_args(idx, L, k_gate, k_out, eps, GANN_VISITED_FAST);
    a.next_query = reinterpret_cast<uint32_t*>(base);  // this call's own counter
    a.stats = nullptr;  // concurrent calls do not touch the index
    a.queries = dq;
    a.nq = nq;
    a.out_ids = k_out ? dids : nullptr;
    a.out_dists = k_out ? dd : nullptr;
    cu(launch_search(a, idx->elem, idx->metric, idx->geom, s), "search kernel");
    if (k_out) {
      cu(cudaMemcpyAsync(h_ids, dids, uint64_t(nq) * k_out * 4, cudaMemcpyDeviceToHost, s), "download ids");
      cu(cudaMemcpyAsync(h_dists, dd, uint64_t(nq) * k_out * 4, cudaMemcpyDeviceToHost, s), "download dists");
    }
  });
}

int gann_alpha_prune(gann_index* idx, const uint32_t* p, const uint64_t* offsets, uint32_t count,
                     const uint32_t* cand_ids, const float* cand_dists, float alpha, int rule,
                     uint32_t* out, uint32_t* n_out) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    if (idx->R == 0) fail(GANN_EINVAL, "degree bound must be positive");  // prune.cpp:11
    check_prune_params(alpha, rule);
    if (count == 0) return;
    set_device(idx);
    const uint64_t total = offsets[count];
    std::vector<uint32_t> len(count), small, big;
    std::vector<uint64_t> beg(count);
    for (uint32_t i = 0; i < count; i++) {
      if (offsets[i + 1] < offsets[i]) fail(GANN_EINVAL, "offsets must be non-decreasing");
      beg[i] = offsets[i];
      const uint64_t m = offsets[i + 1] - offsets[i];
      if (m >= 0xFFFFFFFFull) fail(GANN_EINVAL, "candidate list too long");
      len[i] = static_cast<uint32_t>(m);
      if (p[i] >= idx->n) fail(GANN_EINVAL, "point id out of range");
      (m <= kPruneSmallCap ? small : big).push_back(i);
    }
    for (uint64_t i = 0; i < total; i++)
      if (cand_ids[i] >= idx->n) fail(GANN_EINVAL, "candidate id out of range");
    // A candidate list is a visited set or a merged row: distinct ids (copies
    // of p are dropped anyway, src/prune.cpp:16-18). The kernels' rank sort
    // needs distinct keys, so a repeated id is rejected rather than guessed at.
    {
      std::vector<uint32_t> tmp;
      for (uint32_t i = 0; i < count; i++) {
        tmp.clear();
        for (uint64_t j = offsets[i]; j < offsets[i + 1]; j++)
          if (cand_ids[j] != p[i]) tmp.push_back(cand_ids[j]);
        std::sort(tmp.begin(), tmp.end());
        if (std::adjacent_find(tmp.begin(), tmp.end()) != tmp.end())
          fail(GANN_EINVAL, "candidate list " + std::to_string(i) + " repeats an id");
      }
    }
    // one scratch block: p | beg | len | small | big | ids | dists | out | nout
    idx->pt.ensure(size_t(count) * 4 * 4 + size_t(count) * 8 + total * 8 + size_t(count) * idx->R * 4 + 64);
    uint8_t* base = idx->pt.as<uint8_t>();
    uint64_t* d_beg = reinterpret_cast<uint64_t*>(base);
    uint32_t* d_p = reinterpret_cast<uint32_t*>(d_beg + count);
    uint32_t* d_len = d_p + count;
    uint32_t* d_small = d_len + count;
    uint32_t* d_big = d_small + count;
    uint32_t* d_ids = d_big + count;
    float* d_d = reinterpret_cast<float*>(d_ids + total);
    uint32_t* d_out = reinterpret_cast<uint32_t*>(d_d + total);
    idx->ps.ensure(size_t(count) * 4);
    uint32_t* d_nout = idx->ps.as<uint32_t>();
    auto h2d = [&](void* dst, const void* src, size_t bytes) {
      if (bytes) cu(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, idx->stream), "upload");
    };
    h2d(d_beg, beg.data(), size_t(count) * 8);
    h2d(d_p, p, size_t(count) * 4);
    h2d(d_len, len.data(), size_t(count) * 4);
    h2d(d_small, small.data(), small.size() * 4);
    h2d(d_big, big.data(), big.size() * 4);
    h2d(d_ids, cand_ids, total * 4);
    h2d(d_d, cand_dists, total * 4);
    cu(cudaMemsetAsync(idx->flags, 0, 8, idx->stream), "memset");
    PruneArgs a = base_prune_args(idx, alpha, rule);
    a.points = d_p;
    a.begins = d_beg;
    a.lengths = d_len;
    a.cand_ids = d_ids;
    a.cand_dists = d_d;
    a.out_rows = d_out;
    a.n_out = d_nout;
    if (!small.empty()) {
      a.count = static_cast<uint32_t>(small.size());
      a.list_index = d_small;
      prune_binned(idx, a, kPruneSmallCap);
    }
    if (!big.empty()) {
      a.count = static_cast<uint32_t>(big.size());
      a.list_index = d_big;
      a.mmin = 0;
      a.mcap = 0xFFFFFFFFu;
      cu(launch_prune(a, idx->elem, idx->metric, idx->geom, 256, idx->stream), "prune kernel");
    }
    cu(cudaMemcpyAsync(out, d_out, size_t(count) * idx->R * 4, cudaMemcpyDeviceToHost, idx->stream), "download");
    if (n_out) cu(cudaMemcpyAsync(n_out, d_nout, size_t(count) * 4, cudaMemcpyDeviceToHost, idx->stream), "download");
    sync(idx);
  });
}

int gann_group_by_key(const uint32_t* keys, const uint32_t* vals, uint64_t m, int device,
                      uint32_t* out_keys, uint32_t* out_vals, uint64_t* offsets, uint64_t* n_groups) {
  return guarded([&] {
    if (n_groups) *n_groups = 0;
    if (m == 0) {
      if (offsets) offsets[0] = 0;
      return;
    }
    if (m >= 0x7FFFFFFFull) fail(GANN_EINVAL, "group_by_key: too many pairs");
    for (uint64_t i = 0; i < m; i++)
      if (keys[i] == GANN_NONE) fail(GANN_EINVAL, "key 0xFFFFFFFF is reserved");
    uint32_t tbits = 6;
    while ((uint64_t(1) << tbits) < 2 * m) tbits++;
    // keys -> dense slots of a device hash table; the slots play the role of
    // target vertices for the counting group-by
    gann_index* idx = new_index(uint64_t(1) << tbits, 1, GANN_U8, GANN_L2, 1, device);
    try {
      idx->pt.ensure(m * 4);
      idx->ps.ensure(m * 4);
      idx->ok.ensure(m * 4);
      idx->ov.ensure(m * 4);
      idx->misc.ensure((size_t(1) << tbits) * 4);
      idx->qids.ensure(m * 4);
      cu(cudaMemcpyAsync(idx->qids.p, keys, m * 4, cudaMemcpyHostToDevice, idx->stream), "upload");
      cu(cudaMemcpyAsync(idx->ps.p, vals, m * 4, cudaMemcpyHostToDevice, idx->stream), "upload");
      cu(launch_hash_keys(idx->qids.as<uint32_t>(), m, idx->misc.as<uint32_t>(), tbits,
                          idx->pt.as<uint32_t>(), idx->stream), "hash keys");
      // a key with more pairs than the counting group-by orders in one block:
      // a stable radix sort of (slot, input index) instead (semisort.cpp:15-73
      // keeps input order inside a group; group order is unspecified)
      uint64_t maxg = 0;
      {
        std::unordered_map<uint32_t, uint64_t> cnt;
        cnt.reserve(m);
        for (uint64_t i = 0; i < m; i++) maxg = std::max(maxg, ++cnt[keys[i]]);
      }
      if (maxg > kSortedGroupCap) {
        std::vector<uint32_t> iota(m);
        for (uint64_t i = 0; i < m; i++) iota[i] = static_cast<uint32_t>(i);
        idx->ok.ensure(m * 4);
        idx->ov.ensure(m * 4);
        cu(cudaMemcpyAsync(idx->ps.p, iota.data(), m * 4, cudaMemcpyHostToDevice, idx->stream), "upload");
        void* tmp = nullptr;
        size_t tmp_bytes = 0;
        const cudaError_t e = stable_sort_pairs_u32(idx->pt.as<uint32_t>(), idx->ok.as<uint32_t>(),
                                                    idx->ps.as<uint32_t>(), idx->ov.as<uint32_t>(), m,
                                                    static_cast<int>(tbits), &tmp, &tmp_bytes, idx->stream);
        std::vector<uint32_t> perm(m);
        if (e == cudaSuccess)
          cu(cudaMemcpyAsync(perm.data(), idx->ov.p, m * 4, cudaMemcpyDeviceToHost, idx->stream), "download");
        cudaStreamSynchronize(idx->stream);
        if (tmp) cudaFree(tmp);
        cu(e, "stable radix sort");
        uint64_t g = 0;
        for (uint64_t j = 0; j < m; j++) {
          out_keys[j] = keys[perm[j]];
          out_vals[j] = vals[perm[j]];
          if (j == 0 || out_keys[j] != out_keys[j - 1]) {
            if (offsets) offsets[g] = j;
            g++;
          }
        }
        if (offsets) offsets[g] = m;
        if (n_groups) *n_groups = g;
        gann_index_free(idx);
        return;
      }
      uint64_t ng = 0;
      apply_back(idx, nullptr, 0, idx->pt.as<uint32_t>(), idx->ps.as<uint32_t>(), m, 1.0f, 0, false,
                 idx->ok.as<uint32_t>(), idx->ov.as<uint32_t>(), &ng, idx->misc.as<uint32_t>());
      cu(cudaMemcpyAsync(out_keys, idx->ok.p, m * 4, cudaMemcpyDeviceToHost, idx->stream), "download");
      cu(cudaMemcpyAsync(out_vals, idx->ov.p, m * 4, cudaMemcpyDeviceToHost, idx->stream), "download");
      sync(idx);
      uint64_t g = 0;
      for (uint64_t i = 0; i < m; i++)
        if (i == 0 || out_keys[i] != out_keys[i - 1]) {
          if (offsets) offsets[g] = i;
          g++;
        }
      if (offsets) offsets[g] = m;
      if (g != ng) fail(GANN_ECUDA, "group count mismatch");
      if (n_groups) *n_groups = g;
    } catch (...) {
      gann_index_free(idx);
      throw;
    }
    gann_index_free(idx);
  });
}

int gann_choose_start(gann_index* idx, uint32_t* start) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    set_device(idx);
    *start = choose_start_dev(idx);
  });
}

int gann_insert_batch(gann_index* idx, const uint32_t* ids, uint32_t count, uint32_t L, float alpha,
                      int rule, uint32_t* back) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    if (L == 0 || idx->R == 0) fail(GANN_EINVAL, "build beam and degree bound must be positive");
    check_prune_params(alpha, rule);
    if (count == 0) return;
    for (uint32_t i = 0; i < count; i++)
      if (ids[i] >= idx->n) fail(GANN_EINVAL, "point id out of range");
    set_device(idx);
    idx->pt.ensure(size_t(count) * 4);
    cu(cudaMemcpyAsync(idx->pt.p, ids, size_t(count) * 4, cudaMemcpyHostToDevice, idx->stream), "upload");
    insert_batch(idx, idx->pt.as<uint32_t>(), count, L, alpha, rule, false);
    if (back) {
      for (uint32_t i = 0; i < count; i++)
        cu(cudaMemcpyAsync(back + size_t(i) * idx->R, idx->adj + uint64_t(ids[i]) * idx->R,
                           size_t(idx->R) * 4, cudaMemcpyDeviceToHost, idx->stream), "download");
      sync(idx);
    }
  });
}

int gann_apply_back_edges(gann_index* idx, const uint32_t* targets, const uint32_t* sources,
                          uint64_t m, float alpha, int rule) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    check_prune_params(alpha, rule);
    if (m == 0) return;
    for (uint64_t i = 0; i < m; i++) {
      if (targets[i] >= idx->n || sources[i] >= idx->n) fail(GANN_EINVAL, "pair id out of range");
      if (targets[i] == sources[i]) fail(GANN_EINVAL, "self loop at vertex " + std::to_string(targets[i]));
    }
    // A repeated (target, source) pair changes nothing after its first
    // occurrence (builder_common.cpp:124-128, first occurrence wins), so it is
    // dropped here, keeping the input order: the sources of a target are then
    // distinct, which is what the group merge needs for groups of any size
    // (a group too large to sort by ordinal always overflows R and is
    // re-pruned, where pair order does not matter).
    std::vector<uint32_t> t2, s2;
    {
      std::vector<uint64_t> seen;
      seen.reserve(m);
      for (uint64_t i = 0; i < m; i++) seen.push_back((uint64_t(targets[i]) << 32) | sources[i]);
      std::vector<uint64_t> sorted = seen;
      std::sort(sorted.begin(), sorted.end());
      if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end()) {
        std::unordered_set<uint64_t> first;
        first.reserve(m * 2);
        for (uint64_t i = 0; i < m; i++)
          if (first.insert(seen[i]).second) {
            t2.push_back(targets[i]);
            s2.push_back(sources[i]);
          }
        targets = t2.data();
        sources = s2.data();
        m = t2.size();
      }
    }
    set_device(idx);
    idx->pt.ensure(m * 4);
    idx->ps.ensure(m * 4);
    cu(cudaMemcpyAsync(idx->pt.p, targets, m * 4, cudaMemcpyHostToDevice, idx->stream), "upload");
    cu(cudaMemcpyAsync(idx->ps.p, sources, m * 4, cudaMemcpyHostToDevice, idx->stream), "upload");
    apply_back(idx, nullptr, 0, idx->pt.as<uint32_t>(), idx->ps.as<uint32_t>(), m, alpha, rule, false, nullptr,
               nullptr, nullptr, nullptr, nullptr, 1, true);
  });
}

int gann_groundtruth_device(gann_index* idx, const void* d_queries, uint32_t nq, uint32_t k,
                            uint32_t* d_ids, float* d_dists, void* stream) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    set_device(idx);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : idx->stream;
    const uint8_t* q = static_cast<const uint8_t*>(d_queries);
    if (idx->stride != idx->row_bytes) {
      idx->q.ensure(size_t(nq) * idx->stride);
      cu(cudaMemsetAsync(idx->q.p, 0, size_t(nq) * idx->stride, s), "memset");
      cu(cudaMemcpy2DAsync(idx->q.p, idx->stride, d_queries, idx->row_bytes, idx->row_bytes, nq,
                           cudaMemcpyDeviceToDevice, s), "stage queries");
      q = idx->q.as<uint8_t>();
    }
    run_groundtruth(idx, q, nq, k, d_ids, d_dists, s);
  });
}

int gann_groundtruth(gann_index* idx, const void* queries, uint32_t nq, uint32_t k, uint32_t* ids,
                     float* dists) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    if (nq == 0) return;
    set_device(idx);
    idx->qids.ensure(size_t(nq) * k * 4);
    idx->qdists.ensure(size_t(nq) * k * 4);
    const uint8_t* q = stage_rows(idx, idx->q, queries, nq, false);
    run_groundtruth(idx, q, nq, k, idx->qids.as<uint32_t>(), idx->qdists.as<float>(), idx->stream);
    cu(cudaMemcpyAsync(ids, idx->qids.p, size_t(nq) * k * 4, cudaMemcpyDeviceToHost, idx->stream), "download");
    cu(cudaMemcpyAsync(dists, idx->qdists.p, size_t(nq) * k * 4, cudaMemcpyDeviceToHost, idx->stream), "download");
    sync(idx);
  });
}

int gann_generate_u8(void* d_out, uint64_t n, uint32_t d, uint32_t clusters, float sigma,
                     float noise_frac, uint64_t center_seed, uint64_t stream_seed, uint64_t row0,
                     int device) {
  return guarded([&] {
    if (clusters == 0 || d == 0) fail(GANN_EINVAL, "gen: d and clusters must be positive");
    cu(cudaSetDevice(device), "cudaSetDevice");
    cu(launch_generate_u8(static_cast<uint8_t*>(d_out), d, n, d, clusters, sigma, noise_frac,
                          center_seed, stream_seed, row0, nullptr),
       "generate");
    cu(cudaDeviceSynchronize(), "generate sync");
  });
}

int gann_normal_table(float* out) {
  return guarded([&] {
    if (!out) fail(GANN_EINVAL, "NULL argument");
    normal_table(out);
  });
}

int gann_generate_f32(void* d_out, uint64_t n, uint32_t d, uint32_t clusters, float sigma, float norm_sigma,
                      float shift, uint64_t center_seed, uint64_t stream_seed, uint64_t row0, int device) {
  return guarded([&] {
    if (clusters == 0 || d == 0) fail(GANN_EINVAL, "gen: d and clusters must be positive");
    cu(cudaSetDevice(device), "cudaSetDevice");
    cu(launch_generate_f32(static_cast<float*>(d_out), n, d, clusters, sigma, norm_sigma, shift, center_seed,
                           stream_seed, row0, nullptr),
       "generate");
    cu(cudaDeviceSynchronize(), "generate sync");
  });
}

void gann_shuffle_swap_log(uint32_t n, uint64_t seed, uint32_t* log) { shuffle_swap_log(n, seed, log); }

void gann_shuffled_order(uint32_t n, uint64_t seed, uint32_t front, uint32_t* out) {
  std::vector<uint32_t> order(n);
  for (uint32_t i = 0; i < n; i++) order[i] = i;
  std::mt19937_64 rng(seed);
  std::shuffle(order.begin(), order.end(), rng);
  if (n) std::iter_swap(order.begin(), std::find(order.begin(), order.end(), front));
  std::copy(order.begin(), order.end(), out);
}

uint32_t gann_batch_ranges(uint64_t n, uint32_t max_batch, uint32_t* lo, uint32_t* hi,
                           uint32_t max_ranges) {
  auto r = batch_ranges(n, max_batch);
  for (size_t i = 0; i < r.size() && i < max_ranges; i++) {
    lo[i] = r[i].first;
    hi[i] = r[i].second;
  }
  return static_cast<uint32_t>(r.size());
}

uint64_t gann_insert_seed(uint64_t seed) { return mix64(seed, 0x696e73657274ULL); }

namespace {

[[noreturn]] void fmt_fail(const std::string& msg) { fail(GANN_EIO, msg); }

void read_exact(std::ifstream& in, void* dst, size_t bytes, const std::string& what) {
  in.read(static_cast<char*>(dst), static_cast<std::streamsize>(bytes));
  if (static_cast<size_t>(in.gcount()) != bytes) fmt_fail("truncated " + what);
}

bool ends_with(const std::string& s, const char* suf) {
  const size_t n = std::strlen(suf);
  return s.size() >= n && s.compare(s.size() - n, n, suf) == 0;
}

}  // namespace

int gann_save_graph(const gann_index* cidx, const char* path) {
  return guarded([&] {
    gann_index* idx = const_cast<gann_index*>(cidx);
    if (!idx || !path) fail(GANN_EINVAL, "NULL argument");
    if (idx->part_count != 1) fail(GANN_EINVAL, "save_graph needs the whole graph (export each partition instead)");
    set_device(idx);
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) fail(GANN_EIO, std::string("cannot open for writing: ") + path);
    const uint64_t n = idx->n;
    const uint32_t R = idx->R;
    out.write("ANNG", 4);
    const uint32_t header[4] = {1u, static_cast<uint32_t>(n), R, idx->start};
    out.write(reinterpret_cast<const char*>(header), sizeof(header));
    // degrees then ids, streamed from the device in slabs
    const uint64_t slab = 1u << 20;
    std::vector<uint32_t> rows(std::min<uint64_t>(n, slab) * R);
    std::vector<uint32_t> deg(n);
    for (int pass = 0; pass < 2; pass++) {
      for (uint64_t v0 = 0; v0 < n; v0 += slab) {
        const uint64_t cnt = std::min<uint64_t>(slab, n - v0);
        cu(cudaMemcpyAsync(rows.data(), idx->adj + v0 * R, cnt * R * 4, cudaMemcpyDeviceToHost, idx->stream),
           "download graph");
        sync(idx);
        for (uint64_t i = 0; i < cnt; i++) {
          const uint32_t* r = rows.data() + i * R;
          uint32_t k = 0;
          while (k < R && r[k] != GANN_NONE) k++;
          if (pass == 0) deg[v0 + i] = k;
          else out.write(reinterpret_cast<const char*>(r), static_cast<std::streamsize>(k) * 4);
        }
      }
      if (pass == 0) out.write(reinterpret_cast<const char*>(deg.data()), static_cast<std::streamsize>(n) * 4);
    }
    if (!out) fail(GANN_EIO, std::string("write failed: ") + path);
  });
}

int gann_load_graph(gann_index* idx, const char* path) {
  return guarded([&] {
    if (!idx || !path) fail(GANN_EINVAL, "NULL argument");
    if (idx->part_count != 1) fail(GANN_EINVAL, "load_graph needs an unpartitioned index");
    const std::string ctx(path);
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(GANN_EIO, "cannot open for reading: " + ctx);
    char magic[4];
    read_exact(in, magic, 4, "graph data: " + ctx);
    if (std::memcmp(magic, "ANNG", 4) != 0) fmt_fail("not a graph file: " + ctx);
    uint32_t header[4];
    read_exact(in, header, sizeof(header), "graph data: " + ctx);
    if (header[0] != 1u) fmt_fail("unsupported graph version " + std::to_string(header[0]) + ": " + ctx);
    const uint32_t n = header[1], cap = header[2], start = header[3];
    if (n > 0 && start >= n) fmt_fail("start vertex out of range: " + ctx);
    if (n != idx->n) fail(GANN_EINVAL, "graph has " + std::to_string(n) + " vertices, index " + std::to_string(idx->n));
    if (cap > idx->R) fail(GANN_EINVAL, "graph capacity " + std::to_string(cap) + " exceeds the index's R");
    std::vector<uint32_t> deg(n);
    read_exact(in, deg.data(), size_t(n) * 4, "graph data: " + ctx);
    std::vector<uint32_t> adj(size_t(n) * idx->R, GANN_NONE), tmp;
    for (uint32_t v = 0; v < n; v++) {
      if (deg[v] > cap) fmt_fail("degree exceeds capacity at vertex " + std::to_string(v) + ": " + ctx);
      uint32_t* r = adj.data() + size_t(v) * idx->R;
      read_exact(in, r, size_t(deg[v]) * 4, "graph data: " + ctx);
      tmp.assign(r, r + deg[v]);
      std::sort(tmp.begin(), tmp.end());
      for (uint32_t t = 0; t < deg[v]; t++) {  // set_neighbors + check_graph_invariants
        if (tmp[t] >= n) fmt_fail("neighbor id out of range at vertex " + std::to_string(v) + ": " + ctx);
        if (tmp[t] == v) fmt_fail("self loop at vertex " + std::to_string(v) + ": " + ctx);
        if (t > 0 && tmp[t] == tmp[t - 1]) fmt_fail("duplicate neighbor at vertex " + std::to_string(v) + ": " + ctx);
      }
    }
    in.peek();
    if (!in.eof()) fmt_fail("trailing bytes: " + ctx);
    set_device(idx);
    if (n) cu(cudaMemcpyAsync(idx->adj, adj.data(), adj.size() * 4, cudaMemcpyHostToDevice, idx->stream), "upload graph");
    if (n) cu(cudaMemsetAsync(idx->spre, 0, n, idx->stream), "clear row prefixes");
    idx->start = start;
    sync(idx);
  });
}

int gann_index_create_from_file(const char* path, int metric, uint32_t R, int device, gann_index** out) {
  int rc = GANN_OK;
  std::vector<uint8_t> payload;
  uint32_t n = 0, d = 0;
  int elem = GANN_F32;
  rc = guarded([&] {
    if (!path || !out) fail(GANN_EINVAL, "NULL argument");
    const std::string p(path);
    // graphann::elem_from_path / format_from_path (src/dataset.cpp:56-66)
    if (ends_with(p, ".fvecs") || ends_with(p, ".fbin")) elem = GANN_F32;
    else if (ends_with(p, ".bvecs") || ends_with(p, ".u8bin")) elem = GANN_U8;
    else if (ends_with(p, ".i8bin")) elem = GANN_I8;
    const size_t esz = elem == GANN_F32 ? 4 : 1;
    const bool vecs = ends_with(p, "vecs");
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) fail(GANN_EIO, "cannot open for reading: " + p);
    const uint64_t fsize = static_cast<uint64_t>(in.tellg());
    in.seekg(0);
    if (!vecs) {
      uint32_t h[2];
      read_exact(in, h, 8, "vector data: " + p);
      n = h[0];
      d = h[1];
      if (n == 0 || d == 0) fmt_fail("empty dataset (n or d is zero): " + p);
      if (fsize != uint64_t(n) * d * esz + 8) fmt_fail("size mismatch (header says " + std::to_string(n) + "x" + std::to_string(d) + "): " + p);
      payload.resize(size_t(n) * d * esz);
      read_exact(in, payload.data(), payload.size(), "vector data: " + p);
    } else {
      read_exact(in, &d, 4, "vector data: " + p);
      if (d == 0) fmt_fail("zero dimension prefix: " + p);
      const uint64_t rec = 4 + uint64_t(d) * esz;
      if (fsize % rec != 0) fmt_fail("truncated or misaligned vecs file: " + p);
      n = static_cast<uint32_t>(fsize / rec);
      payload.resize(size_t(n) * d * esz);
      read_exact(in, payload.data(), d * esz, "vector data: " + p);
      for (uint32_t i = 1; i < n; i++) {
        uint32_t di = 0;
        read_exact(in, &di, 4, "vector data: " + p);
        if (di != d) fmt_fail("inconsistent dimension prefix at vector " + std::to_string(i) + ": " + p);
        read_exact(in, payload.data() + size_t(i) * d * esz, d * esz, "vector data: " + p);
      }
    }
  });
  if (rc != GANN_OK) return rc;
  return gann_index_create(payload.data(), n, d, elem, metric, R, device, out);
}

int gann_range_search(gann_index* idx, const void* queries, uint32_t nq, float radius, uint32_t L,
                      float eps, uint32_t cap, uint32_t* counts, uint32_t* ids, float* dists) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    if (!(radius > 0)) fail(GANN_EINVAL, "range radius must be positive");  // search.cpp:136
    validate_search(idx, 0, L, L, eps, GANN_VISITED_FAST);
    if (nq == 0) return;
    // internal_radius (src/dataset.cpp:248-250): squared under l2, as is under ip
    const float rr = idx->metric == GANN_L2 ? radius * radius : radius;
    uint32_t vcap = 4 * L + 64;
    std::vector<uint32_t> vi, nv(nq);
    std::vector<float> vd;
    for (int attempt = 0; attempt < 4; attempt++) {
      vi.assign(size_t(nq) * vcap, GANN_NONE);
      vd.assign(size_t(nq) * vcap, 0.0f);
      const int rc = gann_search(idx, queries, nq, 0, L, L, eps, GANN_VISITED_FAST, nullptr, nullptr, nullptr,
                                 nv.data(), nullptr, vi.data(), vd.data(), vcap);
      if (rc != GANN_OK) fail(rc, g_err);
      const uint32_t vmax = *std::max_element(nv.begin(), nv.end());
      if (vmax <= vcap) break;
      vcap = vmax;  // a long walk: run again with room for every visited vertex
    }
    for (uint32_t q = 0; q < nq; q++) {
      std::vector<std::pair<float, uint32_t>> in;
      for (uint32_t t = 0; t < nv[q]; t++) {
        const float dv = vd[size_t(q) * vcap + t];
        if (dv <= rr) in.emplace_back(dv, vi[size_t(q) * vcap + t]);
      }
      std::sort(in.begin(), in.end());  // (dist, id): neighbor_less
      counts[q] = static_cast<uint32_t>(in.size());
      for (uint32_t t = 0; t < cap; t++) {
        const bool have = t < in.size();
        if (ids) ids[size_t(q) * cap + t] = have ? in[t].second : GANN_NONE;
        if (dists) dists[size_t(q) * cap + t] = have ? in[t].first : __builtin_inff();
      }
    }
  });
}

// ---- vertex-partitioned build ---------------------------------------------------
int gann_index_create_part(const void* points, uint64_t n, uint32_t d, int elem, int metric, uint32_t R,
                           uint32_t rank, uint32_t nparts, int device, gann_index** out) {
  return guarded([&] {
    if (!out || (n && !points)) fail(GANN_EINVAL, "NULL argument");
    gann_index* idx = new_index(n, d, elem, metric, R, device, rank, nparts);
    try {
      if (n)
        cu(cudaMemcpy2DAsync(idx->points, idx->stride, points, idx->row_bytes, idx->row_bytes, n,
                             cudaMemcpyHostToDevice, idx->stream),
           "upload points");
      sync(idx);
    } catch (...) {
      gann_index_free(idx);
      throw;
    }
    *out = idx;
  });
}

int gann_index_create_part_device(const void* d_points, uint64_t n, uint32_t d, int elem, int metric, uint32_t R,
                                  uint32_t rank, uint32_t nparts, int device, gann_index** out) {
  return guarded([&] {
    if (!out) fail(GANN_EINVAL, "NULL argument");
    gann_index* idx = new_index(n, d, elem, metric, R, device, rank, nparts);
    try {
      // d_points NULL: the points stay zero for the caller to write in place
      // (gann_index_device_ptrs) — at 1B points a second copy would not fit
      if (n && d_points)
        cu(cudaMemcpy2DAsync(idx->points, idx->stride, d_points, idx->row_bytes, idx->row_bytes, n,
                             cudaMemcpyDeviceToDevice, idx->stream),
           "copy points");
      sync(idx);
    } catch (...) {
      gann_index_free(idx);
      throw;
    }
    *out = idx;
  });
}

int gann_part_info(const gann_index* idx, uint32_t* rank, uint32_t* nparts, uint64_t* base, uint64_t* rows) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    if (rank) *rank = idx->part_rank;
    if (nparts) *nparts = idx->part_count;
    if (base) *base = idx->part_base;
    if (rows) *rows = idx->part_rows;
  });
}

int gann_part_ipc_handle(const gann_index* idx, void* handle64) {
  return guarded([&] {
    if (!idx || !handle64) fail(GANN_EINVAL, "NULL argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cu(cudaSetDevice(idx->device), "cudaSetDevice");
    cudaIpcMemHandle_t h;
    cu(cudaIpcGetMemHandle(&h, idx->adj), "cudaIpcGetMemHandle");
    std::memcpy(handle64, &h, 64);
  });
}

int gann_part_attach(gann_index* idx, uint32_t rank, const void* handle64) {
  return guarded([&] {
    if (!idx || !handle64) fail(GANN_EINVAL, "NULL argument");
    if (rank >= idx->part_count) fail(GANN_EINVAL, "partition rank out of range");
    if (rank == idx->part_rank) return;  // our own rows
    set_device(idx);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    void* ptr = nullptr;
    cu(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    idx->ipc_open.push_back(ptr);
    uint32_t* row0 = static_cast<uint32_t*>(ptr);
    cu(cudaMemcpy(idx->d_parts + rank, &row0, sizeof(row0), cudaMemcpyHostToDevice), "parts table");
  });
}

int gann_part_build_begin(gann_index* idx, uint32_t L, float alpha, int rule, uint64_t seed, uint32_t max_batch,
                          uint32_t* nbatches) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    if (idx->n == 0) fail(GANN_EINVAL, "cannot build over an empty dataset");
    if (L == 0 || idx->R == 0) fail(GANN_EINVAL, "build beam and degree bound must be positive");
    check_prune_params(alpha, rule);
    set_device(idx);
    const uint64_t n = idx->n;
    cu(cudaMemsetAsync(idx->adj, 0xFF, uint64_t(idx->part_rows) * idx->R * 4, idx->stream), "clear graph");
    cu(cudaMemsetAsync(idx->spre, 0, std::max<uint64_t>(idx->part_rows, 1), idx->stream), "clear row prefixes");
    cu(cudaMemsetAsync(idx->tcount, 0, uint64_t(idx->part_rows) * 4, idx->stream), "clear counts");
    // every partition derives the same start and insertion order (src/diskann.cpp:47-51)
    idx->start = choose_start_dev(idx);
    idx->order_host.resize(n);
    gann_shuffled_order(static_cast<uint32_t>(n), mix64(seed, 0x696e73657274ULL), idx->start, idx->order_host.data());
    idx->order.ensure(n * 4);
    cu(cudaMemcpyAsync(idx->order.p, idx->order_host.data(), n * 4, cudaMemcpyHostToDevice, idx->stream), "order");
    idx->ranges = batch_ranges(n, max_batch);
    idx->bL = L;
    idx->balpha = alpha;
    idx->brule = static_cast<uint32_t>(rule);
    sync(idx);
    if (nbatches) *nbatches = static_cast<uint32_t>(idx->ranges.size());
  });
}

namespace {
// Phase 1 of a partitioned batch: insert the batch points this partition owns,
// then emit their reverse pairs grouped by the target's owner (counts[g]
// pairs for partition g, at *d_pairs in partition order).
void part_phase1(gann_index* idx, uint32_t batch, uint64_t* counts, const uint32_t** d_pairs) {
    if (batch >= idx->ranges.size()) fail(GANN_EINVAL, "batch index out of range");
    set_device(idx);
    const auto [lo, hi] = idx->ranges[batch];
    // this partition's points of the batch (owner(v) = v / P) and their batch offsets
    std::vector<uint32_t> ids, bo;
    for (uint32_t pos = lo; pos < hi; pos++) {
      const uint32_t v = idx->order_host[pos];
      if (v / idx->part_size == idx->part_rank) {
        ids.push_back(v);
        bo.push_back(pos - lo);
      }
    }
    const uint32_t K = static_cast<uint32_t>(ids.size());
    const uint32_t G = idx->part_count;
    idx->lids.ensure(size_t(K) * 8 + 16);
    uint32_t* d_ids = idx->lids.as<uint32_t>();
    uint32_t* d_bo = d_ids + K;
    if (K) {
      cu(cudaMemcpyAsync(d_ids, ids.data(), size_t(K) * 4, cudaMemcpyHostToDevice, idx->stream), "upload");
      cu(cudaMemcpyAsync(d_bo, bo.data(), size_t(K) * 4, cudaMemcpyHostToDevice, idx->stream), "upload");
      insert_batch(idx, d_ids, K, idx->bL, idx->balpha, static_cast<int>(idx->brule), true);
    }
    // reverse pairs (target, batch ordinal), grouped by the target's owner
    idx->pair_cnt.ensure(sizeof(unsigned long long) * 2 * G);
    unsigned long long* d_cnt = idx->pair_cnt.as<unsigned long long>();
    cu(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * G, idx->stream), "memset");
    cu(part_pairs_count(idx->adj, idx->part_base, idx->R, d_ids, K, idx->part_size, d_cnt, idx->stream), "pairs");
    std::vector<unsigned long long> cnt(G), off(G);
    cu(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(unsigned long long) * G, cudaMemcpyDeviceToHost, idx->stream), "read");
    sync(idx);
    unsigned long long total = 0;
    for (uint32_t g = 0; g < G; g++) {
      off[g] = total;
      total += cnt[g];
      counts[g] = cnt[g];
    }
    idx->pair_out.ensure(std::max<unsigned long long>(total, 1) * 8);
    cu(cudaMemcpyAsync(d_cnt + G, off.data(), sizeof(unsigned long long) * G, cudaMemcpyHostToDevice, idx->stream),
       "offsets");
    cu(part_pairs_scatter(idx->adj, idx->part_base, idx->R, d_ids, d_bo, K, idx->part_size, d_cnt + G,
                          idx->pair_out.as<uint32_t>(), idx->stream),
       "pairs");
    sync(idx);
    *d_pairs = idx->pair_out.as<uint32_t>();
}

// Phase 2: merge the m received pairs (interleaved target, batch ordinal).
void part_phase2(gann_index* idx, uint32_t batch, const uint32_t* d_pairs, uint64_t m) {
    if (batch >= idx->ranges.size()) fail(GANN_EINVAL, "batch index out of range");
    set_device(idx);
    const auto [lo, hi] = idx->ranges[batch];
    // the received pairs carry their batch ordinal: the merge sorts by it, which
    // restores the single-GPU pair order (src/diskann.cpp:61-65) inside each group
    apply_back(idx, idx->order.as<uint32_t>() + lo, hi - lo, d_pairs, nullptr, m, idx->balpha,
               static_cast<int>(idx->brule), true, nullptr, nullptr, nullptr, nullptr, d_pairs + 1, 2);
    sync(idx);
}

void xcheck(int rc, const char* what) {
  if (rc != 0) fail(GANN_ECUDA, std::string("exchange ") + what + " failed (rc " + std::to_string(rc) + ")");
}
}  // namespace

int gann_part_phase1(gann_index* idx, uint32_t batch, uint64_t* counts, const uint32_t** d_pairs) {
  return guarded([&] {
    if (!idx || !counts || !d_pairs) fail(GANN_EINVAL, "NULL argument");
    part_phase1(idx, batch, counts, d_pairs);
  });
}

int gann_part_phase2(gann_index* idx, uint32_t batch, const uint32_t* d_pairs, uint64_t m) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    part_phase2(idx, batch, d_pairs, m);
  });
}

int gann_part_batch_cap(const gann_index* idx, uint32_t L, uint64_t budget_bytes, uint32_t* max_batch) {
  return guarded([&] {
    if (!idx || !max_batch) fail(GANN_EINVAL, "NULL argument");
    if (L == 0) fail(GANN_EINVAL, "build beam must be positive");
    // per point of a global batch, on one of G ranks: its 1/G share of the
    // inserts (visited ids + dists of 3L slots, counters, bins, pair output)
    // and of the received reverse pairs (<= R per point, 1.5x for skew across
    // owners): the pair itself, the group-by arrays and the merged lists at
    // ~0.25 groups per pair (measured 0.22 at 10M) of R + 1 slots each
    const double G = idx->part_count, R = idx->R;
    const uint32_t vcap = std::max<uint32_t>(64, 3 * L);
    const double insert = 8.0 * vcap + 48.0 + 8.0 * R;
    const double per_pair = 8.0 + 4.0 + 4.0 + 0.25 * 40.0 + (0.25 * R + 1.0) * 8.0;
    const double per_point = (insert + 1.5 * R * per_pair) / G;
    const double fixed = double(1ull << 30) + 64.0 * (1 << 20);  // prune hand-off + small buffers
    const double room = double(budget_bytes) - fixed;
    const double cap = room > 0 ? room / per_point : 0.0;
    *max_batch = static_cast<uint32_t>(std::min(cap, double(idx->n)));
    if (*max_batch == 0) fail(GANN_EINVAL, "budget leaves no room for a build batch");
  });
}

// The whole partitioned build in C++: build_diskann's batch loop
// (src/diskann.cpp:53-67) with one exchange step per batch. The collectives
// are the caller's (gann_exchange): NCCL through gann_exchange_nccl, or any
// transport with the same semantics (the tests use torch.distributed/gloo).
int gann_part_build(gann_index* idx, const gann_exchange* x, uint32_t L, float alpha, int rule, uint64_t seed,
                    uint32_t max_batch, uint64_t* pairs_sent) {
  const int rc0 = gann_part_build_begin(idx, L, alpha, rule, seed, max_batch, nullptr);
  if (rc0 != GANN_OK) return rc0;
  return guarded([&] {
    if (!x || !x->alltoall_counts || !x->alltoallv || !x->barrier) fail(GANN_EINVAL, "incomplete exchange");
    if (x->rank != idx->part_rank || x->nranks != idx->part_count)
      fail(GANN_EINVAL, "exchange rank/size differ from the index's partition");
    const uint32_t G = idx->part_count;
    std::vector<uint64_t> sc(G), rc(G);
    uint64_t sent = 0;
    for (uint32_t b = 0; b < idx->ranges.size(); b++) {
      const uint32_t* d_send = nullptr;
      part_phase1(idx, b, sc.data(), &d_send);
      xcheck(x->alltoall_counts(x->ctx, sc.data(), rc.data()), "counts");
      uint64_t m = 0;
      for (uint32_t g = 0; g < G; g++) m += rc[g], sent += sc[g];
      idx->pair_in.ensure(std::max<uint64_t>(m, 1) * 8);
      xcheck(x->alltoallv(x->ctx, d_send, sc.data(), idx->pair_in.p, rc.data(), idx->stream), "pairs");
      cu(cudaStreamSynchronize(idx->stream), "exchange sync");
      part_phase2(idx, b, idx->pair_in.as<uint32_t>(), m);
      // every partition's rows are final before the next batch's searches read them
      xcheck(x->barrier(x->ctx, idx->stream), "barrier");
    }
    idx->pair_in.release();
    if (pairs_sent) *pairs_sent = sent;
  });
}

// ---- layered (HNSW) search: search_hnsw, src/hnsw.cpp:130-147 ---------------
// Layer 0 is an ordinary index (points + bottom graph). The upper layers are
// graphs over the same id space (non-members have empty rows), held on the
// device beside it. A query descends with beam {1, 1, 0} searches from the
// entry vertex, layer by layer, each started at the previous layer's nearest
// (start_override, in place on the device), then runs the bottom search from
// there; dist_comps is the sum over all layers.
struct gann_hnsw {
  gann_index* base = nullptr;  // borrowed
  uint32_t layers = 1;
  uint32_t m = 0;              // upper-layer row capacity
  uint32_t entry = 0;
  uint32_t* upper = nullptr;   // (layers - 1) x n x m
  DevBuf cur, dc, hd;
};

int gann_hnsw_create(gann_index* layer0, uint32_t num_layers, const uint32_t* upper_adj, uint32_t m_upper,
                     uint32_t entry, gann_hnsw** out) {
  return guarded([&] {
    if (!layer0 || !out) fail(GANN_EINVAL, "NULL argument");
    if (num_layers == 0) fail(GANN_EINVAL, "an HNSW index has at least one layer");
    if (layer0->part_count != 1) fail(GANN_EINVAL, "layered search over a partitioned index is not supported");
    const uint64_t n = layer0->n;
    if (n && entry >= n) fail(GANN_EINVAL, "entry vertex out of range");
    if (num_layers > 1) {
      if (m_upper == 0 || m_upper > 1024) fail(GANN_EINVAL, "upper-layer capacity must lie in [1, 1024]");
      if (!upper_adj) fail(GANN_EINVAL, "upper_adj is NULL");
    }
    set_device(layer0);
    auto* h = new gann_hnsw();
    h->base = layer0;
    h->layers = num_layers;
    h->m = num_layers > 1 ? m_upper : 0;
    h->entry = entry;
    if (num_layers > 1 && n) {
      const size_t bytes = size_t(num_layers - 1) * n * m_upper * 4;
      if (cudaMalloc(&h->upper, bytes) != cudaSuccess) {
        delete h;
        fail(GANN_ECUDA, "cudaMalloc upper layers");
      }
      cu(cudaMemcpy(h->upper, upper_adj, bytes, cudaMemcpyHostToDevice), "upload upper layers");
      try {
        for (uint32_t l = 1; l < num_layers; l++)
          validate_graph_rows(layer0, h->upper + uint64_t(l - 1) * n * m_upper, n, m_upper, n, 0,
                              "layer " + std::to_string(l) + ": ");
      } catch (...) {
        cudaFree(h->upper);
        delete h;
        throw;
      }
    }
    *out = h;
  });
}

void gann_hnsw_free(gann_hnsw* h) {
  if (!h) return;
  cudaSetDevice(h->base->device);
  if (h->base->stream) cudaStreamSynchronize(h->base->stream);
  if (h->upper) cudaFree(h->upper);
  for (DevBuf* b : {&h->cur, &h->dc, &h->hd}) b->release();
  delete h;
}

int gann_hnsw_search(gann_hnsw* h, const void* queries, uint32_t nq, uint32_t k_out, uint32_t L, uint32_t k_gate,
                     float eps, int visited_mode, uint32_t* ids, float* dists, uint32_t* n_visited,
                     uint64_t* dist_comps) {
  return guarded([&] {
    if (!h) fail(GANN_EINVAL, "index is NULL");
    gann_index* idx = h->base;
    validate_search(idx, k_out, L, k_gate, eps, visited_mode);
    if (nq == 0) return;
    if (!queries) fail(GANN_EINVAL, "queries is NULL");
    set_device(idx);
    if (idx->n == 0) {  // src/hnsw.cpp:134 — empty index, empty result
      for (uint64_t i = 0; i < uint64_t(nq) * k_out; i++) {
        if (ids) ids[i] = GANN_NONE;
        if (dists) dists[i] = __builtin_inff();
      }
      for (uint32_t i = 0; i < nq; i++) {
        if (n_visited) n_visited[i] = 0;
        if (dist_comps) dist_comps[i] = 0;
      }
      return;
    }
    const uint8_t* q = stage_rows(idx, idx->q, queries, nq, false);
    h->cur.ensure(size_t(nq) * 4);
    h->dc.ensure(size_t(nq) * 8 * h->layers);
    h->hd.ensure(size_t(nq) * 4);
    uint32_t* cur = h->cur.as<uint32_t>();
    uint64_t* dc = h->dc.as<uint64_t>();
    {
      std::vector<uint32_t> e(nq, h->entry);
      cu(cudaMemcpyAsync(cur, e.data(), size_t(nq) * 4, cudaMemcpyHostToDevice, idx->stream), "upload entry");
      sync(idx);  // e leaves scope
    }
    // upper layers, top down: beam {1, 1, 0} from cur, the nearest found becomes cur
    for (uint32_t l = h->layers - 1; l >= 1; l--) {
      SearchArgs a = base_search_args(idx, 1, 1, 1, 0.0f, visited_mode);
      a.graph = GraphView{h->upper + size_t(l - 1) * idx->n * h->m, nullptr, 0, 1, 0};
      a.R = h->m;
      a.queries = q;
      a.nq = nq;
      a.start_override = cur;
      a.out_ids = cur;  // a query reads its start before it writes its result
      a.out_dists = h->hd.as<float>();
      a.dist_comps = dc + size_t(l) * nq;
      run_search(idx, a, idx->stream);
    }
    SearchArgs a = base_search_args(idx, L, k_gate, k_out, eps, visited_mode);
    a.queries = q;
    a.nq = nq;
    a.start_override = cur;
    if (k_out) {
      idx->qids.ensure(size_t(nq) * k_out * 4);
      idx->qdists.ensure(size_t(nq) * k_out * 4);
      a.out_ids = idx->qids.as<uint32_t>();
      a.out_dists = idx->qdists.as<float>();
    }
    idx->qnvis.ensure(size_t(nq) * 4);
    a.n_visited = idx->qnvis.as<uint32_t>();
    a.dist_comps = dc;
    run_search(idx, a, idx->stream);
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
      if (dst) cu(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, idx->stream), "download results");
    };
    if (k_out) {
      d2h(ids, a.out_ids, size_t(nq) * k_out * 4);
      d2h(dists, a.out_dists, size_t(nq) * k_out * 4);
    }
    d2h(n_visited, a.n_visited, size_t(nq) * 4);
    std::vector<uint64_t> all(dist_comps ? size_t(nq) * h->layers : 0);
    if (dist_comps) d2h(all.data(), dc, all.size() * 8);
    sync(idx);
    if (dist_comps)
      for (uint32_t i = 0; i < nq; i++) {
        uint64_t t = 0;
        for (uint32_t l = 0; l < h->layers; l++) t += all[size_t(l) * nq + i];
        dist_comps[i] = t;
      }
  });
}

int gann_get_stats(const gann_index* idx, gann_stats* out) {
  return guarded([&] {
    if (!idx || !out) fail(GANN_EINVAL, "NULL argument");
    cudaSetDevice(idx->device);
    cu(cudaDeviceSynchronize(), "device sync");  // launches on any stream have counted
    unsigned long long slots[kStCount * kStatSlots], s[kStCount] = {};
    cu(cudaMemcpy(slots, idx->stats, sizeof(slots), cudaMemcpyDeviceToHost), "read stats");
    for (uint32_t t = 0; t < kStatSlots; t++)
      for (uint32_t i = 0; i < kStCount; i++) s[i] += slots[t * kStCount + i];
    out->queries = s[kStQueries];
    out->expansions = s[kStExpansions];
    out->evaluations = s[kStEvals];
    out->filter_drops = s[kStDrops];
    out->adj_entries = s[kStAdj];
    out->prune_lists = s[kStPruneLists];
    out->prune_candidates = s[kStPruneCands];
    out->prune_evals = s[kStPruneEvals];
    out->merges = s[kStMerges];
    out->survivors = s[kStSurvivors];
    out->moved = s[kStMoved];
    out->duplicates = s[kStDups];
    out->guess_hits = s[kStGuess];
    out->back_pairs = idx->back_pairs;
    out->back_groups = idx->back_groups;
    out->back_pruned = idx->back_pruned;
    for (int i = 0; i < 6; i++) out->build_ms[i] = idx->build_ms[i];
  });
}

int gann_reset_stats(gann_index* idx) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    set_device(idx);
    // launches queued on other streams (any caller stream) count before the reset
    cu(cudaDeviceSynchronize(), "device sync");
    cu(cudaMemsetAsync(idx->stats, 0, sizeof(unsigned long long) * kStCount * kStatSlots, idx->stream), "memset");
    sync(idx);
  });
}

int gann_index_device_ptrs(const gann_index* idx, void** points, uint64_t* stride, uint32_t** adj) {
  return guarded([&] {
    if (!idx) fail(GANN_EINVAL, "index is NULL");
    if (points) *points = idx->points;
    if (stride) *stride = idx->stride;
    if (adj) *adj = idx->adj;
  });
}

}  // extern "C"
