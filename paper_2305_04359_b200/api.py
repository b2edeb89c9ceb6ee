"""Host-side mirror of the reference's hot-path interface, over the C ABI.

Names, argument meaning and error behaviour follow graphann (the reference,
``proj/include/graphann/*.hpp``): ``DiskannParams`` / ``SearchParams`` /
``PruneParams``, ``build_diskann``, ``beam_search``, ``alpha_prune``,
``group_by_key``, ``choose_start``, ``shuffled_order``, ``batch_ranges``,
``insert_point``, ``apply_back_edges``. Where the reference throws
``std::invalid_argument`` this raises ``ValueError``; CUDA failures raise
``GannError``. All compute runs in ``libgann_b200.so`` on the GPU — there is
no CPU path here.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from ._lib import GANN_NONE, GannStats, check, lib

ELEM = {np.dtype(np.uint8): 0, np.dtype(np.int8): 1, np.dtype(np.float32): 2}
ELEM_DTYPE = {0: np.uint8, 1: np.int8, 2: np.float32}
METRIC = {"l2": 0, "ip": 1}
RULE = {"scale_candidate": 0, "scale_selected": 1}
VISITED = {"fast": 0, "ref": 1, "exact": 2}


def _p(a) -> Optional[int]:
    return None if a is None else a.ctypes.data


# ---- parameter blocks (include/graphann/{diskann,search,prune}.hpp) ---------
@dataclass
class DiskannParams:
    """graphann::DiskannParams (include/graphann/diskann.hpp:14-20) + the batch cap."""
    degree_bound: int = 64   # R
    build_beam: int = 128    # L
    alpha: float = 1.2
    rule: str = "scale_candidate"
    seed: int = 42
    max_batch: int = 0       # 0 = the reference's uncapped prefix doubling


@dataclass
class SearchParams:
    """graphann::SearchParams (include/graphann/search.hpp:14-18)."""
    beam: int = 10           # L
    k: int = 10              # results; also the expansion gate
    epsilon: float = 0.0


@dataclass
class PruneParams:
    """graphann::PruneParams (include/graphann/prune.hpp:20-24)."""
    degree_bound: int = 64
    alpha: float = 1.2
    rule: str = "scale_candidate"


@dataclass
class SearchResult:
    """Batched graphann::SearchResult (include/graphann/search.hpp:40-44)."""
    ids: np.ndarray                  # (nq, k) uint32, GANN_NONE padded, ascending (dist, id)
    dists: np.ndarray                # (nq, k) float32, +inf padded
    n_visited: np.ndarray            # (nq,) |V|
    dist_comps: np.ndarray           # (nq,) distance evaluations
    visited_ids: Optional[np.ndarray] = None    # (nq, vcap) expansion order
    visited_dists: Optional[np.ndarray] = None


@dataclass
class GroupedPairs:
    """graphann::GroupedPairs (include/graphann/semisort.hpp:14-19)."""
    keys: np.ndarray
    vals: np.ndarray
    group_offsets: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint64))

    def groups(self) -> int:
        return max(0, len(self.group_offsets) - 1)


class Index:
    """HBM-resident points + fixed-degree graph (VectorDataset + NeighborGraph)."""

    def __init__(self, points: np.ndarray, metric: str = "l2", degree_bound: int = 64,
                 device: int = 0):
        points = np.ascontiguousarray(points)
        if points.ndim != 2:
            raise ValueError("points must be a 2-d array (n, d)")
        if points.dtype not in ELEM:
            raise ValueError(f"unsupported element type {points.dtype}")
        if metric not in METRIC:
            raise ValueError(f"unknown metric '{metric}' (expected l2 or ip)")
        h = C.c_void_p()
        check(lib().gann_index_create(_p(points), points.shape[0], points.shape[1], ELEM[points.dtype],
                                      METRIC[metric], degree_bound, device, C.byref(h)))
        self._init(h, metric, device)

    @classmethod
    def from_device(cls, ptr: int, n: int, d: int, dtype, metric: str = "l2", degree_bound: int = 64,
                    device: int = 0) -> "Index":
        """Wrap points already in device memory (row-major, d elements per row)."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        check(lib().gann_index_create_device(C.c_void_p(ptr), n, d, ELEM[np.dtype(dtype)], METRIC[metric],
                                             degree_bound, device, C.byref(h)))
        self._init(h, metric, device)
        return self

    def _init(self, h, metric, device):
        self._h = h
        self.metric = metric
        self.device = device
        n, d, e, m, R, s = C.c_uint64(), C.c_uint32(), C.c_int(), C.c_int(), C.c_uint32(), C.c_uint32()
        check(lib().gann_index_info(h, C.byref(n), C.byref(d), C.byref(e), C.byref(m), C.byref(R), C.byref(s)))
        self.n, self.d, self.R = n.value, d.value, R.value
        self.dtype = np.dtype(ELEM_DTYPE[e.value])

    # -- lifetime ---------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().gann_index_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def start(self) -> int:
        s = C.c_uint32()
        check(lib().gann_index_info(self._h, None, None, None, None, None, C.byref(s)))
        return s.value

    # -- build ------------------------------------------------------------------
    def build(self, params: DiskannParams = DiskannParams()) -> "Index":
        if params.degree_bound != self.R:
            raise ValueError(f"index capacity R={self.R} differs from params.degree_bound={params.degree_bound}")
        check(lib().gann_build(self._h, params.build_beam, params.alpha, RULE[params.rule], params.seed,
                               params.max_batch))
        return self

    def import_graph(self, adj: np.ndarray, start: int) -> None:
        adj = np.ascontiguousarray(adj, dtype=np.uint32)
        if adj.shape != (self.n, self.R):
            raise ValueError(f"graph must be ({self.n}, {self.R})")
        check(lib().gann_import_graph(self._h, _p(adj), start))

    def export_graph(self):
        adj = np.empty((self.n, self.R), np.uint32)
        deg = np.empty(self.n, np.uint32)
        s = C.c_uint32()
        check(lib().gann_export_graph(self._h, _p(adj), _p(deg), C.byref(s)))
        return adj, deg, s.value

    @classmethod
    def from_file(cls, path: str, metric: str = "l2", degree_bound: int = 64, device: int = 0) -> "Index":
        """graphann::load_vectors (src/dataset.cpp:71-122): .u8bin/.i8bin/.fbin/.bvecs/.fvecs."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        check(lib().gann_index_create_from_file(str(path).encode(), METRIC[metric], degree_bound, device,
                                                C.byref(h)))
        self._init(h, metric, device)
        return self

    def save_graph(self, path: str) -> None:
        """graphann::save_graph (ANNG, src/graph.cpp:101-121)."""
        check(lib().gann_save_graph(self._h, str(path).encode()))

    def load_graph(self, path: str) -> None:
        """graphann::load_graph (src/graph.cpp:136-178) into this index."""
        check(lib().gann_load_graph(self._h, str(path).encode()))

    def range_search(self, queries: np.ndarray, radius: float, params: SearchParams, cap: int = 256):
        """graphann::range_search (src/search.cpp:133-149), batched: returns a list
        of (ids, dists) per query, ascending (dist, id)."""
        queries = np.ascontiguousarray(queries)
        if queries.ndim != 2 or queries.shape[1] != self.d or queries.dtype != self.dtype:
            raise ValueError("query does not match dataset dimension/element kind")
        nq = queries.shape[0]
        counts = np.empty(nq, np.uint32)
        ids = np.empty((nq, cap), np.uint32)
        dists = np.empty((nq, cap), np.float32)
        check(lib().gann_range_search(self._h, _p(queries), nq, radius, params.beam, params.epsilon, cap,
                                      _p(counts), _p(ids), _p(dists)))
        if (counts > cap).any():
            return self.range_search(queries, radius, params, int(counts.max()))
        return [(ids[i, : counts[i]].copy(), dists[i, : counts[i]].copy()) for i in range(nq)]

    # -- search -----------------------------------------------------------------
    def search(self, queries: np.ndarray, params: SearchParams = SearchParams(), k_out: Optional[int] = None,
               visited_mode: str = "fast", start_override=None, vcap: int = 0) -> SearchResult:
        queries = np.ascontiguousarray(queries)
        if queries.ndim != 2 or queries.shape[1] != self.d or queries.dtype != self.dtype:
            raise ValueError("query does not match dataset dimension/element kind")
        nq = queries.shape[0]
        k_out = params.k if k_out is None else k_out
        ids = np.empty((nq, k_out), np.uint32)
        dists = np.empty((nq, k_out), np.float32)
        nvis = np.empty(nq, np.uint32)
        dc = np.empty(nq, np.uint64)
        vi = np.empty((nq, vcap), np.uint32) if vcap else None
        vd = np.empty((nq, vcap), np.float32) if vcap else None
        so = None if start_override is None else np.ascontiguousarray(start_override, dtype=np.uint32)
        if so is not None and so.shape != (nq,):
            raise ValueError("start_override needs one start per query")
        check(lib().gann_search(self._h, _p(queries), nq, k_out, params.beam, params.k, params.epsilon,
                                VISITED[visited_mode], _p(so), _p(ids), _p(dists), _p(nvis), _p(dc),
                                _p(vi), _p(vd), vcap))
        if vcap:  # entries past |V| are padding
            pad = np.arange(vcap)[None, :] >= nvis[:, None]
            vi[pad] = GANN_NONE
            vd[pad] = np.inf
        return SearchResult(ids, dists, nvis, dc, vi, vd)

    def run_sweep(self, queries: np.ndarray, truth_ids: np.ndarray, truth_dists: np.ndarray, sweep, meta,
                  visited_mode: str = "fast"):
        """graphann::run_sweep (src/eval.cpp:127-168) with this index's batched
        search as the dispatch: one gann_search call over all queries per sweep
        point and repetition (evalutil.run_sweep)."""
        from .evalutil import run_sweep

        def one(beam, k, eps):
            r = self.search(queries, SearchParams(beam, k, eps), k_out=k, visited_mode=visited_mode)
            return r.ids, r.dist_comps
        return run_sweep(one, truth_ids, truth_dists, sweep, meta)

    def search_device(self, q_ptr: int, nq: int, params: SearchParams, k_out: int, ids_ptr: int,
                      dists_ptr: int, nvis_ptr: int = 0, dc_ptr: int = 0, stream: int = 0,
                      visited_mode: str = "fast") -> None:
        check(lib().gann_search_device(self._h, C.c_void_p(q_ptr), nq, k_out, params.beam, params.k,
                                       params.epsilon, VISITED[visited_mode], C.c_void_p(ids_ptr), C.c_void_p(dists_ptr),
                                       C.c_void_p(nvis_ptr or None), C.c_void_p(dc_ptr or None),
                                       C.c_void_p(stream or None)))

    def max_beam(self) -> int:
        """The largest search beam L this index holds on chip (gann_search_max_beam)."""
        v = C.c_uint32(0)
        check(lib().gann_search_max_beam(self._h, C.byref(v)))
        return int(v.value)

    def stage_queries(self, q_ptr: int, nq: int) -> None:
        check(lib().gann_stage_queries(self._h, C.c_void_p(q_ptr), nq))

    def search_staged(self, params: SearchParams, k_out: int, ids_ptr: int, dists_ptr: int,
                      stream: int = 0) -> None:
        check(lib().gann_search_staged(self._h, k_out, params.beam, params.k, params.epsilon,
                                       C.c_void_p(ids_ptr), C.c_void_p(dists_ptr), C.c_void_p(stream or None)))

    def async_scratch_bytes(self, nq: int, k_out: int) -> int:
        return int(lib().gann_search_async_scratch(self._h, nq, k_out))

    def search_async(self, h_queries_ptr: int, nq: int, params: SearchParams, k_out: int, h_ids_ptr: int,
                     h_dists_ptr: int, scratch_ptr: int, scratch_bytes: int, stream: int) -> None:
        """Enqueue a host-buffer search on `stream` (gann_search_async): the H2D
        copy, the kernel and the D2H copy; returns at once. Calls on different
        streams with their own scratch run concurrently."""
        check(lib().gann_search_async(self._h, C.c_void_p(h_queries_ptr), nq, k_out, params.beam, params.k,
                                      params.epsilon, C.c_void_p(h_ids_ptr), C.c_void_p(h_dists_ptr),
                                      C.c_void_p(scratch_ptr), scratch_bytes, C.c_void_p(stream or None)))

    # -- build internals ------------------------------------------------------------
    def alpha_prune_many(self, points, candidate_ids, candidate_dists, params: PruneParams):
        """alpha_prune over many lists; returns a list of kept-id arrays."""
        if params.degree_bound != self.R:
            raise ValueError("params.degree_bound must equal the index capacity R")
        offs = np.zeros(len(points) + 1, np.uint64)
        offs[1:] = np.cumsum([len(c) for c in candidate_ids])
        ids = np.ascontiguousarray(np.concatenate([np.asarray(c, np.uint32) for c in candidate_ids])
                                   if len(points) else np.zeros(0, np.uint32))
        ds = np.ascontiguousarray(np.concatenate([np.asarray(c, np.float32) for c in candidate_dists])
                                  if len(points) else np.zeros(0, np.float32))
        p = np.ascontiguousarray(points, dtype=np.uint32)
        out = np.empty((max(len(p), 1), self.R), np.uint32)
        nout = np.empty(max(len(p), 1), np.uint32)
        check(lib().gann_alpha_prune(self._h, _p(p), _p(offs), len(p), _p(ids), _p(ds), params.alpha,
                                     RULE[params.rule], _p(out), _p(nout)))
        return [out[i, : nout[i]].copy() for i in range(len(p))]

    def choose_start(self) -> int:
        s = C.c_uint32()
        check(lib().gann_choose_start(self._h, C.byref(s)))
        return s.value

    def insert(self, ids, build_beam: int, alpha: float, rule: str = "scale_candidate") -> np.ndarray:
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        back = np.empty((len(ids), self.R), np.uint32)
        check(lib().gann_insert_batch(self._h, _p(ids), len(ids), build_beam, alpha, RULE[rule], _p(back)))
        return back

    def apply_back_edges(self, targets, sources, params: PruneParams) -> None:
        t = np.ascontiguousarray(targets, dtype=np.uint32)
        s = np.ascontiguousarray(sources, dtype=np.uint32)
        if t.shape != s.shape:
            raise ValueError("targets and sources differ in length")
        check(lib().gann_apply_back_edges(self._h, _p(t), _p(s), len(t), params.alpha, RULE[params.rule]))

    def groundtruth(self, queries: np.ndarray, k: int):
        queries = np.ascontiguousarray(queries, dtype=self.dtype)
        nq = queries.shape[0]
        ids = np.empty((nq, k), np.uint32)
        dists = np.empty((nq, k), np.float32)
        check(lib().gann_groundtruth(self._h, _p(queries), nq, k, _p(ids), _p(dists)))
        return ids, dists

    def groundtruth_device(self, q_ptr: int, nq: int, k: int, ids_ptr: int, dists_ptr: int, stream: int = 0):
        check(lib().gann_groundtruth_device(self._h, C.c_void_p(q_ptr), nq, k, C.c_void_p(ids_ptr),
                                            C.c_void_p(dists_ptr), C.c_void_p(stream or None)))

    # -- counters -------------------------------------------------------------------
    def stats(self) -> dict:
        s = GannStats()
        check(lib().gann_get_stats(self._h, C.byref(s)))
        out = {name: getattr(s, name) for name, _ in GannStats._fields_ if name != "build_ms"}
        out["build_ms"] = dict(zip(["start", "search", "prune", "group", "merge", "reprune"], list(s.build_ms)))
        return out

    def reset_stats(self) -> None:
        check(lib().gann_reset_stats(self._h))

    def release_scratch(self) -> None:
        """Free the build's batch scratch (gann_release_scratch)."""
        check(lib().gann_release_scratch(self._h))

    def device_ptrs(self):
        pts, adj = C.c_void_p(), C.c_void_p()
        stride = C.c_uint64()
        check(lib().gann_index_device_ptrs(self._h, C.byref(pts), C.byref(stride), C.byref(adj)))
        return pts.value, stride.value, adj.value


# ---- module-level mirrors of the reference's free functions ------------------------
class HnswIndex:
    """A layered index (graphann::HnswIndex, include/graphann/hnsw.hpp) searched
    on the GPU with graphann::search_hnsw semantics (src/hnsw.cpp:130-147).

    ``layer0`` is an :class:`Index` holding the points and the bottom graph
    (borrowed: keep it alive); ``upper`` lists the graphs of layers 1..top as
    (n, m) id arrays over the same id space (rows of non-members are empty);
    ``entry`` is the top layer's entry vertex. The layers come from a builder
    outside this path (the reference's build_hnsw); the search is the product."""

    def __init__(self, layer0: Index, upper, entry: int):
        self.layer0 = layer0
        upper = [np.ascontiguousarray(a, dtype=np.uint32) for a in upper]
        m = upper[0].shape[1] if upper else 0
        for a in upper:
            if a.shape != (layer0.n, m):
                raise ValueError(f"every upper layer must be ({layer0.n}, {m})")
        flat = np.ascontiguousarray(np.stack(upper)) if upper else None
        h = C.c_void_p()
        check(lib().gann_hnsw_create(layer0.handle, 1 + len(upper), _p(flat), m, entry, C.byref(h)))
        self._h = h
        self.num_layers = 1 + len(upper)
        self.entry = entry

    def close(self):
        if getattr(self, "_h", None):
            lib().gann_hnsw_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search(self, queries: np.ndarray, params: SearchParams = SearchParams(), k_out: Optional[int] = None,
               visited_mode: str = "fast") -> SearchResult:
        queries = np.ascontiguousarray(queries)
        if queries.ndim != 2 or queries.shape[1] != self.layer0.d or queries.dtype != self.layer0.dtype:
            raise ValueError("query does not match dataset dimension/element kind")
        nq = queries.shape[0]
        k_out = params.k if k_out is None else k_out
        ids = np.empty((nq, k_out), np.uint32)
        dists = np.empty((nq, k_out), np.float32)
        nvis = np.empty(nq, np.uint32)
        dc = np.empty(nq, np.uint64)
        check(lib().gann_hnsw_search(self._h, _p(queries), nq, k_out, params.beam, params.k, params.epsilon,
                                     VISITED[visited_mode], _p(ids), _p(dists), _p(nvis), _p(dc)))
        return SearchResult(ids, dists, nvis, dc)


def _hnsw_run_sweep(self, queries, truth_ids, truth_dists, sweep, meta, visited_mode: str = "fast"):
    """run_sweep with search_hnsw as the dispatch (the reference's layered_dispatch)."""
    from .evalutil import run_sweep

    def one(beam, k, eps):
        r = self.search(queries, SearchParams(beam, k, eps), k_out=k, visited_mode=visited_mode)
        return r.ids, r.dist_comps
    return run_sweep(one, truth_ids, truth_dists, sweep, meta)


HnswIndex.run_sweep = _hnsw_run_sweep


def search_hnsw(index: HnswIndex, queries: np.ndarray, params: SearchParams = SearchParams(), **kw) -> SearchResult:
    """graphann::search_hnsw (src/hnsw.cpp:130-147), batched over queries."""
    return index.search(queries, params, **kw)


def build_diskann(points: np.ndarray, metric: str = "l2", params: DiskannParams = DiskannParams(),
                  device: int = 0) -> Index:
    """graphann::build_diskann (include/graphann/diskann.hpp:36-37)."""
    if points.shape[0] == 0:
        raise ValueError("cannot build over an empty dataset")
    idx = Index(points, metric, params.degree_bound, device)
    return idx.build(params)


def beam_search(index: Index, queries: np.ndarray, params: SearchParams = SearchParams(), **kw) -> SearchResult:
    """graphann::beam_search (include/graphann/search.hpp:57-60), batched."""
    return index.search(queries, params, **kw)


def alpha_prune(index: Index, p: int, candidate_ids, candidate_dists, params: PruneParams) -> np.ndarray:
    """graphann::alpha_prune (include/graphann/prune.hpp:31-33) for one list."""
    return index.alpha_prune_many([p], [candidate_ids], [candidate_dists], params)[0]


def group_by_key(keys, vals, device: int = 0) -> GroupedPairs:
    """graphann::group_by_key (include/graphann/semisort.hpp:21-22) on the GPU."""
    k = np.ascontiguousarray(keys, dtype=np.uint32)
    v = np.ascontiguousarray(vals, dtype=np.uint32)
    if k.shape != v.shape:
        raise ValueError("keys and values differ in length")
    m = len(k)
    ok = np.empty(m, np.uint32)
    ov = np.empty(m, np.uint32)
    off = np.empty(m + 1, np.uint64)
    ng = C.c_uint64()
    check(lib().gann_group_by_key(_p(k), _p(v), m, device, _p(ok), _p(ov), _p(off), C.byref(ng)))
    g = ng.value
    return GroupedPairs(ok, ov, off[: g + 1].copy() if m else np.zeros(0, np.uint64))


def choose_start(index: Index) -> int:
    """graphann::choose_start (include/graphann/builder_common.hpp:21)."""
    return index.choose_start()


def shuffled_order(n: int, seed: int, front: int) -> np.ndarray:
    """graphann::shuffled_order (include/graphann/builder_common.hpp:24)."""
    out = np.empty(n, np.uint32)
    lib().gann_shuffled_order(n, seed, front, _p(out))
    return out


def shuffle_swap_log(n: int, seed: int) -> np.ndarray:
    """std::shuffle's swap log for (n, seed) (gann_shuffle_swap_log): element i swaps with log[i]."""
    out = np.empty(n, np.uint32)
    lib().gann_shuffle_swap_log(n, seed, _p(out))
    return out


def insert_seed(seed: int) -> int:
    """The seed build_diskann passes to shuffled_order (src/diskann.cpp:51)."""
    return int(lib().gann_insert_seed(seed))


def batch_ranges(n: int, max_batch: int = 0):
    """graphann::batch_ranges (include/graphann/builder_common.hpp:17) + cap."""
    cap = 64 + (n // max_batch if max_batch else 0)
    lo = np.empty(cap, np.uint32)
    hi = np.empty(cap, np.uint32)
    c = lib().gann_batch_ranges(n, max_batch, _p(lo), _p(hi), cap)
    return [(int(a), int(b)) for a, b in zip(lo[:c], hi[:c])]


def insert_point(index: Index, j: int, build_beam: int, alpha: float, rule: str = "scale_candidate"):
    """graphann::insert_point (include/graphann/diskann.hpp:26-29): returns the
    reverse pairs (q, j) for q in the new out-list."""
    back = index.insert([j], build_beam, alpha, rule)[0]
    return [(int(q), j) for q in back[back != GANN_NONE]]


def apply_back_edges(index: Index, edges, params: PruneParams) -> None:
    """graphann::apply_back_edges (include/graphann/builder_common.hpp:31-34)."""
    e = np.asarray(edges, dtype=np.uint32).reshape(-1, 2)
    index.apply_back_edges(e[:, 0], e[:, 1], params)
