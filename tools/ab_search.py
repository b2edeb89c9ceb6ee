"""A/B timing of search-kernel variants selected by environment variables, on
one GPU-built index (serial launches, CUDA events on the launching stream).

  python tools/ab_search.py --n 10000000 --L 200 --var GANN_SEARCH_DIAG=0
"""
import argparse
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_04359_b200 as g  # noqa: E402
from paper_2305_04359_b200 import datagen  # noqa: E402
from paper_2305_04359_b200._lib import check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--nq", type=int, default=10_000)
ap.add_argument("--L", default="200")
ap.add_argument("--var", action="append", default=[], help="NAME=v1,v2 (repeatable; cartesian product)")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--sort-clusters", action="store_true",
                help="experiment: permute the points so that each mixture cluster is contiguous")
ap.add_argument("--profile", action="store_true", help="one launch per L between cudaProfilerStart/Stop (ncu)")
args = ap.parse_args()

cfg = datagen.CONFIGS[args.config].scaled(args.n)
torch.cuda.set_stream(torch.cuda.Stream())
base = torch.empty(cfg.n * cfg.d, dtype=torch.uint8, device="cuda")
check(lib().gann_generate_u8(base.data_ptr(), cfg.n, cfg.d, cfg.clusters, cfg.sigma, cfg.noise_frac,
                             cfg.center_seed, cfg.base_seed, 0, 0))
q = torch.empty(args.nq * cfg.d, dtype=torch.uint8, device="cuda")
check(lib().gann_generate_u8(q.data_ptr(), args.nq, cfg.d, cfg.clusters, cfg.sigma, cfg.noise_frac,
                             cfg.center_seed, cfg.query_seed, 0, 0))
if args.sort_clusters:
    r = np.arange(cfg.n, dtype=np.uint64)
    c = datagen.mix64_2(np.uint64(cfg.base_seed) ^ datagen.K_CLUSTER, r) % np.uint64(cfg.clusters)
    perm = torch.from_numpy(np.argsort(c, kind="stable").astype(np.int64)).cuda()
    base = base.view(cfg.n, cfg.d)[perm].contiguous().view(-1)
    print("points sorted by cluster", flush=True)
idx = g.Index.from_device(base.data_ptr(), cfg.n, cfg.d, np.uint8, "l2", cfg.R)
idx.build(g.DiskannParams(cfg.R, cfg.L, cfg.alpha, max_batch=cfg.max_batch))
torch.cuda.synchronize()
print("build_ms", {k: round(v, 1) for k, v in idx.stats()["build_ms"].items()}, flush=True)
idx.stage_queries(q.data_ptr(), args.nq)
s = torch.cuda.current_stream()

combos = [{}]
for v in args.var:
    name, vals = v.split("=")
    combos = [dict(c, **{name: x}) for c in combos for x in vals.split(",")]


def run(L, env):
    for k, v in env.items():
        os.environ[k] = v
    ids = torch.empty(args.nq * 10, dtype=torch.int32, device="cuda")
    ds = torch.empty(args.nq * 10, dtype=torch.float32, device="cuda")
    idx.search_staged(g.SearchParams(L, L, 0.0), 10, ids.data_ptr(), ds.data_ptr(), s.cuda_stream)  # warm
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.reps):
        idx.search_staged(g.SearchParams(L, L, 0.0), 10, ids.data_ptr(), ds.data_ptr(), s.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / args.reps, ids.cpu().numpy()


if args.profile:
    for L in [int(x) for x in args.L.split(",")]:
        run(L, combos[0])
        torch.cuda.profiler.start()
        run(L, combos[0])
        torch.cuda.profiler.stop()
    sys.exit(0)

for L in [int(x) for x in args.L.split(",")]:
    res = {i: [] for i in range(len(combos))}
    ref_ids = None
    evq = {}
    stq = {}
    for r in range(args.rounds):
        for i, c in enumerate(combos):
            idx.reset_stats()
            ms, ids = run(L, c)
            st = idx.stats()
            evq[i] = st["evaluations"] / max(1, st["queries"])
            stq[i] = (st["merges"] / max(1, st["queries"]), st["guess_hits"] / max(1, st["expansions"]))
            res[i].append(ms)
            if ref_ids is None:
                ref_ids = ids
            assert (ids == ref_ids).all(), f"ids differ under {c}"
    for i, c in enumerate(combos):
        ms = min(res[i])
        print(f"L={L} {c}: {ms:.3f} ms  {args.nq / ms * 1e3 / 1e6:.3f} MQPS  evals/q {evq[i]:.1f}  steps/q {stq[i][0]:.1f} dropped/exp {stq[i][1]:.3f}  "
              f"(runs {[round(x, 3) for x in res[i]]})")
    # diagnostic counters (general kernel) for the first combo
    os.environ["GANN_SEARCH_DIAG"] = "1"
    for k, v in combos[-1].items():
        os.environ[k] = v
    idx.reset_stats()
    run(L, combos[-1])
    st = idx.stats()
    os.environ["GANN_SEARCH_DIAG"] = "0"
    nq = max(1, st["queries"])
    print(f"L={L} diag: exp/q {st['expansions'] / nq:.1f} evals/q {st['evaluations'] / nq:.1f} "
          f"guess_hits/exp {st['guess_hits'] / max(1, st['expansions']):.3f} dups/q {st['duplicates'] / nq:.1f} "
          f"merges/q {st['merges'] / nq:.1f} survivors/merge {st['survivors'] / max(1, st['merges']):.2f} "
          f"moved/merge {st['moved'] / max(1, st['merges']):.1f}",
          flush=True)
