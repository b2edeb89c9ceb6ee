"""TEST INFRASTRUCTURE — ctypes front end for the two CPU oracles.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or the
CPU baseline: never as the thing measured or shipped.

* ``Oracle("orc")`` — ``oracle/_build/libgann_oracle.so``, the scalar C++
  restatement of the reference hot path (``oracle/gann_oracle.cpp``).
* ``Oracle("ref")`` — ``oracle/_ref/libgraphann_ref.so``, the reference's own
  sources compiled by ``oracle/Makefile`` behind ``oracle/ref_shim.cpp``.

Arrays follow the product's conventions: graphs are ``(n, R)`` uint32 with
0xFFFFFFFF padding, data is ``(n, d)`` of uint8 / int8 / float32.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SENT = 0xFFFFFFFF
ELEM = {np.dtype(np.uint8): 0, np.dtype(np.int8): 1, np.dtype(np.float32): 2}
METRIC = {"l2": 0, "ip": 1}
RULE = {"scale_candidate": 0, "scale_selected": 1}

_LIBS = {
    "orc": HERE / "_build" / "libgann_oracle.so",
    "ref": HERE / "_ref" / "libgraphann_ref.so",
}


def available(prefix: str) -> bool:
    return _LIBS[prefix].exists()


def build(with_ref: bool | None = None) -> None:
    """Compile the oracles (make -C oracle [ref]); the reference leg only when
    its sources are present (this container — GPU boxes use the prebuilt .so)."""
    import subprocess

    if with_ref is None:
        with_ref = Path("/root/reference/proj/src").exists()
    targets = ["all"] + (["ref"] if with_ref else [])
    subprocess.run(["make", "-s", "-C", str(HERE)] + targets, check=True)


class OracleError(RuntimeError):
    pass


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    def __init__(self, prefix: str = "orc"):
        path = _LIBS[prefix]
        if not path.exists():
            raise FileNotFoundError(f"oracle library {path} missing: run `make -C oracle{' ref' if prefix == 'ref' else ''}`")
        self.prefix = prefix
        self.lib = C.CDLL(str(path))
        L = self.lib
        f = lambda name: getattr(L, f"{prefix}_{name}")
        u32, u64, i32, f32, vp = C.c_uint32, C.c_uint64, C.c_int, C.c_float, C.c_void_p
        f("last_error").restype = C.c_char_p
        f("distance").restype = f32
        f("distance").argtypes = [vp, vp, u32, i32, i32]
        f("beam_search").argtypes = [vp, u32, u32, u32, vp, u32, i32, i32, vp, u32, u32, u32, f32,
                                     i32, vp, vp, vp, vp, vp, vp, vp, u32, i32]
        f("alpha_prune").argtypes = [u32, vp, vp, u32, vp, u32, u32, i32, i32, u32, f32, i32, vp, vp, vp]
        f("group_by_key").argtypes = [vp, vp, u64, i32, vp, vp, vp, vp]
        f("choose_start").argtypes = [vp, u32, u32, i32, i32, i32, vp]
        f("shuffled_order").argtypes = [u32, u64, u32, vp]
        f("shuffled_order").restype = None
        f("batch_ranges").argtypes = [u32, u32, vp, vp, u32]
        f("batch_ranges").restype = u32
        f("insert_point").argtypes = [vp, u32, u32, u32, vp, u32, i32, i32, u32, u32, f32, i32, vp, vp]
        f("apply_back_edges").argtypes = [vp, u32, u32, vp, u32, i32, i32, vp, vp, u64, f32, i32, i32]
        f("build").argtypes = [vp, u32, u32, i32, i32, u32, u32, f32, i32, u64, u32, i32, vp, vp]
        f("groundtruth").argtypes = [vp, u32, vp, u32, u32, i32, i32, u32, vp, vp, i32]
        f("time_search").argtypes = [vp, u32, u32, u32, vp, u32, i32, i32, vp, u32, u32, u32, f32, u32, i32,
                                     u32, C.c_double, vp, vp, vp]
        f("range_search").argtypes = [vp, u32, u32, u32, vp, u32, i32, i32, vp, u32, f32, u32, f32, u32, vp, vp, vp]
        f("save_graph").argtypes = [vp, u32, u32, u32, C.c_char_p]
        f("load_graph").argtypes = [C.c_char_p, vp, vp, vp, vp, u64]
        if prefix == "ref":
            L.ref_write_vectors.argtypes = [vp, u32, u32, i32, C.c_char_p, i32]
            L.ref_hnsw_build.argtypes = [vp, u32, u32, i32, i32, u32, u32, f32, i32, u64, i32, i32, vp, vp, vp]
            L.ref_hnsw_export.argtypes = [u32, u32, vp, vp, vp]
            L.ref_hnsw_search.argtypes = [u32, vp, u32, u32, i32, i32, vp, u32, u32, u32, f32, vp, vp, vp, vp,
                                          vp, u32, i32]
            L.ref_hnsw_free.argtypes = [u32]
            d64 = C.c_double
            L.ref_pareto.argtypes = [u32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
            L.ref_write_csv.argtypes = [C.c_char_p, C.c_char_p, u32, d64, u64, u32, vp, vp, vp, vp, vp, vp, vp,
                                        C.c_char_p]
            L.ref_hnsw_free.restype = None
        f("recall").restype = C.c_double
        f("recall").argtypes = [vp, vp, u32, vp, u32, u32]
        self._f = f

    def _check(self, rc):
        if rc != 0:
            msg = self._f("last_error")().decode()
            if rc == 1:
                raise ValueError(msg)
            raise OracleError(f"{self.prefix} rc={rc}: {msg}")

    # ---- hot-path functions -------------------------------------------------
    def distance(self, a, b, metric="l2"):
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        return float(self._f("distance")(_p(a), _p(b), a.shape[-1], ELEM[a.dtype], METRIC[metric]))

    def beam_search(self, adj, start, data, queries, L, k, eps=0.0, metric="l2", visited_mode=0,
                    start_override=None, vcap=0, workers=1):
        adj = np.ascontiguousarray(adj, dtype=np.uint32)
        data = np.ascontiguousarray(data)
        queries = np.ascontiguousarray(queries, dtype=data.dtype)
        n, R = adj.shape
        nq = queries.shape[0]
        ids = np.empty((nq, k), np.uint32)
        dists = np.empty((nq, k), np.float32)
        nvis = np.empty(nq, np.uint32)
        dc = np.empty(nq, np.uint64)
        vi = np.full((nq, vcap), SENT, np.uint32) if vcap else None
        vd = np.full((nq, vcap), np.inf, np.float32) if vcap else None
        so = None if start_override is None else np.ascontiguousarray(start_override, dtype=np.uint32)
        self._check(self._f("beam_search")(_p(adj), n, R, start, _p(data), data.shape[1], ELEM[data.dtype],
                                           METRIC[metric], _p(queries), nq, L, k, eps, visited_mode, _p(so),
                                           _p(ids), _p(dists), _p(nvis), _p(dc), _p(vi), _p(vd), vcap, workers))
        out = dict(ids=ids, dists=dists, n_visited=nvis, dist_comps=dc)
        if vcap:
            out.update(visited_ids=vi, visited_dists=vd)
        return out

    def alpha_prune(self, p, ids, dists, data, R, alpha, rule="scale_candidate", metric="l2"):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        dists = np.ascontiguousarray(dists, dtype=np.float32)
        data = np.ascontiguousarray(data)
        out = np.empty(max(R, 1), np.uint32)
        nout = np.zeros(1, np.uint32)
        dc = np.zeros(1, np.uint64)
        self._check(self._f("alpha_prune")(p, _p(ids), _p(dists), len(ids), _p(data), data.shape[0],
                                           data.shape[1], ELEM[data.dtype], METRIC[metric], R, alpha,
                                           RULE[rule], _p(out), _p(nout), _p(dc)))
        return out[: int(nout[0])].copy(), int(dc[0])

    def group_by_key(self, keys, vals, workers=1):
        keys = np.ascontiguousarray(keys, dtype=np.uint32)
        vals = np.ascontiguousarray(vals, dtype=np.uint32)
        m = len(keys)
        ok = np.empty(m, np.uint32)
        ov = np.empty(m, np.uint32)
        off = np.zeros(m + 1, np.uint64)
        ng = np.zeros(1, np.uint64)
        self._check(self._f("group_by_key")(_p(keys), _p(vals), m, workers, _p(ok), _p(ov), _p(off), _p(ng)))
        g = int(ng[0])
        return ok, ov, off[: g + 1] if m else np.zeros(0, np.uint64)

    def choose_start(self, data, metric="l2", workers=1):
        data = np.ascontiguousarray(data)
        s = np.zeros(1, np.uint32)
        self._check(self._f("choose_start")(_p(data), data.shape[0], data.shape[1], ELEM[data.dtype],
                                            METRIC[metric], workers, _p(s)))
        return int(s[0])

    def shuffled_order(self, n, seed, front):
        out = np.empty(n, np.uint32)
        self._f("shuffled_order")(n, seed, front, _p(out))
        return out

    def batch_ranges(self, n, cap=0):
        lo = np.empty(64 + (n // max(cap, 1) if cap else 0), np.uint32)
        hi = np.empty_like(lo)
        c = self._f("batch_ranges")(n, cap, _p(lo), _p(hi), len(lo))
        return [(int(a), int(b)) for a, b in zip(lo[:c], hi[:c])]

    def insert_point(self, adj, start, data, j, L, alpha, rule="scale_candidate", metric="l2"):
        adj = np.array(adj, dtype=np.uint32, order="C")
        data = np.ascontiguousarray(data)
        n, R = adj.shape
        back = np.empty(R, np.uint32)
        nb = np.zeros(1, np.uint32)
        self._check(self._f("insert_point")(_p(adj), n, R, start, _p(data), data.shape[1], ELEM[data.dtype],
                                            METRIC[metric], j, L, alpha, RULE[rule], _p(back), _p(nb)))
        return adj, back[: int(nb[0])].copy()

    def apply_back_edges(self, adj, data, targets, sources, alpha, rule="scale_candidate", metric="l2",
                         workers=1):
        adj = np.array(adj, dtype=np.uint32, order="C")
        data = np.ascontiguousarray(data)
        t = np.ascontiguousarray(targets, dtype=np.uint32)
        s = np.ascontiguousarray(sources, dtype=np.uint32)
        n, R = adj.shape
        self._check(self._f("apply_back_edges")(_p(adj), n, R, _p(data), data.shape[1], ELEM[data.dtype],
                                                METRIC[metric], _p(t), _p(s), len(t), alpha, RULE[rule], workers))
        return adj

    def build(self, data, R, L, alpha, rule="scale_candidate", metric="l2", seed=42, cap=0, workers=0):
        data = np.ascontiguousarray(data)
        n = data.shape[0]
        adj = np.empty((n, R), np.uint32)
        s = np.zeros(1, np.uint32)
        self._check(self._f("build")(_p(data), n, data.shape[1], ELEM[data.dtype], METRIC[metric], R, L,
                                     alpha, RULE[rule], seed, cap, workers, _p(adj), _p(s)))
        return adj, int(s[0])

    def groundtruth(self, data, queries, k, metric="l2", workers=0):
        data = np.ascontiguousarray(data)
        queries = np.ascontiguousarray(queries, dtype=data.dtype)
        nq = queries.shape[0]
        ids = np.empty((nq, k), np.uint32)
        dists = np.empty((nq, k), np.float32)
        self._check(self._f("groundtruth")(_p(data), data.shape[0], _p(queries), nq, data.shape[1],
                                           ELEM[data.dtype], METRIC[metric], k, _p(ids), _p(dists), workers))
        return ids, dists

    def time_search(self, adj, start, data, queries, L, k, eps=0.0, k_out=10, metric="l2", workers=0,
                    reps=3, min_seconds=0.0):
        """Best-of-reps wall seconds for one pass over the queries (measure_qps),
        plus the first pass's top-k_out ids."""
        adj = np.ascontiguousarray(adj, dtype=np.uint32)
        data = np.ascontiguousarray(data)
        queries = np.ascontiguousarray(queries, dtype=data.dtype)
        n, R = adj.shape
        nq = queries.shape[0]
        ids = np.empty((nq, k_out), np.uint32)
        best = np.zeros(1, np.float64)
        done = np.zeros(1, np.uint32)
        self._check(self._f("time_search")(_p(adj), n, R, start, _p(data), data.shape[1], ELEM[data.dtype],
                                           METRIC[metric], _p(queries), nq, L, k, eps, k_out, workers, reps,
                                           min_seconds, _p(ids), _p(best), _p(done)))
        return float(best[0]), ids, int(done[0])

    def range_search(self, adj, start, data, queries, radius, L, eps=0.0, metric="l2", cap=256):
        adj = np.ascontiguousarray(adj, dtype=np.uint32)
        data = np.ascontiguousarray(data)
        queries = np.ascontiguousarray(queries, dtype=data.dtype)
        n, R = adj.shape
        nq = len(queries)
        counts = np.empty(nq, np.uint32)
        ids = np.empty((nq, cap), np.uint32)
        dists = np.empty((nq, cap), np.float32)
        self._check(self._f("range_search")(_p(adj), n, R, start, _p(data), data.shape[1], ELEM[data.dtype],
                                            METRIC[metric], _p(queries), nq, radius, L, eps, cap, _p(counts),
                                            _p(ids), _p(dists)))
        return [(ids[i, : min(counts[i], cap)].copy(), dists[i, : min(counts[i], cap)].copy())
                for i in range(nq)], counts

    def save_graph(self, adj, start, path):
        adj = np.ascontiguousarray(adj, dtype=np.uint32)
        self._check(self._f("save_graph")(_p(adj), adj.shape[0], adj.shape[1], start, str(path).encode()))

    def load_graph(self, path):
        n, cap, s = np.zeros(1, np.uint32), np.zeros(1, np.uint32), np.zeros(1, np.uint32)
        self._check(self._f("load_graph")(str(path).encode(), _p(n), _p(cap), _p(s), None, 0))
        adj = np.empty((int(n[0]), int(cap[0])), np.uint32)
        self._check(self._f("load_graph")(str(path).encode(), _p(n), _p(cap), _p(s), _p(adj), adj.size))
        return adj, int(s[0])

    def write_vectors(self, data, path, fmt="bin"):
        data = np.ascontiguousarray(data)
        self._check(self.lib.ref_write_vectors(_p(data), data.shape[0], data.shape[1], ELEM[data.dtype],
                                               str(path).encode(), 0 if fmt == "bin" else 1))

    # ---- layered (HNSW) index: the reference's build_hnsw / search_hnsw ------
    def hnsw_build(self, data, m, ef, alpha=1.2, rule="scale_candidate", metric="l2", seed=42,
                   single_layer=False, workers=0):
        """graphann::build_hnsw; returns (handle, levels, entry, layers) where
        layers[l] is the (n, cap_l) row array of layer l (0 = bottom)."""
        data = np.ascontiguousarray(data)
        n = data.shape[0]
        h, nl, e = (np.zeros(1, np.uint32) for _ in range(3))
        self._check(self.lib.ref_hnsw_build(_p(data), n, data.shape[1], ELEM[data.dtype], METRIC[metric], m, ef,
                                            alpha, RULE[rule], seed, int(single_layer), workers, _p(h), _p(nl),
                                            _p(e)))
        nl = int(nl[0])
        cap = 2 * m
        levels = np.empty(n, np.uint32)
        caps = np.empty(nl, np.uint32)
        adj = np.empty((nl, n, cap), np.uint32)
        self._check(self.lib.ref_hnsw_export(int(h[0]), cap, _p(levels), _p(caps), _p(adj)))
        layers = [np.ascontiguousarray(adj[l, :, :int(caps[l])]) for l in range(nl)]
        return int(h[0]), levels, int(e[0]), layers

    def hnsw_search(self, handle, data, queries, L, k, eps=0.0, metric="l2", vcap=0, workers=0):
        data = np.ascontiguousarray(data)
        queries = np.ascontiguousarray(queries, dtype=data.dtype)
        nq = queries.shape[0]
        ids = np.empty((nq, k), np.uint32)
        dists = np.empty((nq, k), np.float32)
        nvis = np.empty(nq, np.uint32)
        dc = np.empty(nq, np.uint64)
        vi = np.full((nq, vcap), SENT, np.uint32) if vcap else None
        self._check(self.lib.ref_hnsw_search(handle, _p(data), data.shape[0], data.shape[1], ELEM[data.dtype],
                                             METRIC[metric], _p(queries), nq, L, k, eps, _p(ids), _p(dists),
                                             _p(nvis), _p(dc), _p(vi), vcap, workers))
        out = dict(ids=ids, dists=dists, n_visited=nvis, dist_comps=dc)
        if vcap:
            out["visited_ids"] = vi
        return out

    def hnsw_free(self, handle):
        self.lib.ref_hnsw_free(handle)

    # ---- eval harness -----------------------------------------------------------
    @staticmethod
    def _row_arrays(rows):
        return (np.array([r.beam for r in rows], np.uint32), np.array([r.k for r in rows], np.uint32),
                np.array([r.epsilon for r in rows], np.float32), np.array([r.recall for r in rows], np.float64),
                np.array([r.qps for r in rows], np.float64), np.array([r.latency_ms for r in rows], np.float64),
                np.array([r.dist_comps for r in rows], np.float64))

    def pareto(self, rows):
        """graphann::pareto_frontier; returns (beam, k, eps, recall, qps) tuples."""
        a = self._row_arrays(rows)
        n = len(rows)
        no = np.zeros(1, np.uint32)
        outs = [np.empty(n, np.uint32), np.empty(n, np.uint32), np.empty(n, np.float32), np.empty(n, np.float64),
                np.empty(n, np.float64)]
        self._check(self.lib.ref_pareto(n, *[_p(x) for x in a], _p(no), *[_p(x) for x in outs]))
        m = int(no[0])
        return [(int(outs[0][i]), int(outs[1][i]), float(outs[2][i]), float(outs[3][i]), float(outs[4][i]))
                for i in range(m)]

    def write_csv(self, meta, rows, path):
        a = self._row_arrays(rows)
        self._check(self.lib.ref_write_csv(meta.algorithm.encode(), meta.dataset.encode(), meta.n, meta.build_seconds,
                                           meta.threads, len(rows), *[_p(x) for x in a], str(path).encode()))

    def recall(self, truth_ids, truth_dists, result, k):
        ti = np.ascontiguousarray(truth_ids, dtype=np.uint32)
        td = np.ascontiguousarray(truth_dists, dtype=np.float32)
        r = np.ascontiguousarray(result, dtype=np.uint32)
        return float(self._f("recall")(_p(ti), _p(td), len(ti), _p(r), len(r), k))

    def mean_recall(self, truth_ids, truth_dists, results, k):
        return float(np.mean([self.recall(truth_ids[i], truth_dists[i], results[i][results[i] != SENT], k)
                              for i in range(len(results))]))


def degrees(adj):
    adj = np.asarray(adj)
    return (adj != SENT).sum(axis=1)
