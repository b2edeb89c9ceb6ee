"""Layered (HNSW) search measured beside the reference:
graphann's build_hnsw makes the layers on the host (setup, untimed), then the
same queries go through gann_hnsw_search (host buffers: H2D + all layers + D2H
per call) and through graphann's search_hnsw on all host threads. One JSON line.

  python tools/bench_hnsw.py --n 100000 --d 128 --Ls 10,20,50,100
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2305_04359_b200 as g  # noqa: E402
from paper_2305_04359_b200 import datagen, evalutil  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402  (the reference: layers + CPU baseline)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c0")
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--nq", type=int, default=10_000)
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--ef", type=int, default=64)
ap.add_argument("--Ls", default="10,20,50,100")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()

cfg = datagen.CONFIGS[args.config].scaled(args.n)
data = datagen.host_base(cfg)
qs = datagen.host_queries(cfg, args.nq)
ref = Oracle("ref")
cores = os.cpu_count()
t0 = time.perf_counter()
h, levels, entry, layers = ref.hnsw_build(data, args.m, args.ef, alpha=cfg.alpha, workers=0)
ref_build_s = time.perf_counter() - t0
tid, td = ref.groundtruth(data, qs, 10, workers=0)
idx0 = g.Index(data, "l2", layers[0].shape[1])
idx0.import_graph(layers[0], entry)
hn = g.HnswIndex(idx0, layers[1:], entry)
points = []
for L in [int(x) for x in args.Ls.split(",")]:
    sp = g.SearchParams(L, L, 0.0)  # Alg. 1: the gate at L, top-10 reported
    r = hn.search(qs, sp, k_out=10)  # warm-up
    best = float("inf")
    for _ in range(args.reps):
        t0 = time.perf_counter()
        r = hn.search(qs, sp, k_out=10)
        best = min(best, time.perf_counter() - t0)
    want = ref.hnsw_search(h, data, qs, L, L, 0.0, workers=0)  # warm-up + ids
    t0 = time.perf_counter()
    want = ref.hnsw_search(h, data, qs, L, L, 0.0, workers=0)
    ref_s = time.perf_counter() - t0
    want["ids"] = want["ids"][:, :10]
    rec = float(evalutil.recall_at_k(tid, td, r.ids, 10).mean())
    points.append({"L": L, "k_gate": L, "recall@10": round(rec, 5), "qps": round(args.nq / best, 1),
                   "reference_qps": round(args.nq / ref_s, 1),
                   "ids_identical_to_reference": float((r.ids == want["ids"]).all(axis=1).mean()),
                   "dist_comps_per_query": round(float(r.dist_comps.mean()), 1)})
ref.hnsw_free(h)
print(json.dumps({
    "metric": "layered (HNSW) search QPS, search_hnsw {L, L, 0}, top-10",
    "unit": "queries/s", "n": args.n, "d": cfg.d, "dtype": cfg.dtype, "queries": args.nq,
    "layers": len(layers), "m": args.m, "ef_construction": args.ef,
    "timing": f"gann_hnsw_search with host buffers (H2D, every layer, D2H), best of {args.reps}; reference: "
              f"graphann search_hnsw, parallel_for over {cores} host threads, one pass",
    "reference_build_s": round(ref_build_s, 2), "points": points}), flush=True)
