"""Distribution of per-query work (|V| and evaluations) on the c1 index, and
how the first-ranked queries' cost relates to the query order (tail study).

  python tools/query_cost.py --n 10000000 --L 200
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_04359_b200 as g  # noqa: E402
from paper_2305_04359_b200 import datagen  # noqa: E402
from paper_2305_04359_b200._lib import check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--nq", type=int, default=10_000)
ap.add_argument("--L", type=int, default=200)
args = ap.parse_args()
cfg = datagen.CONFIGS["c1"].scaled(args.n)
base = torch.empty(cfg.n * cfg.d, dtype=torch.uint8, device="cuda")
check(lib().gann_generate_u8(base.data_ptr(), cfg.n, cfg.d, cfg.clusters, cfg.sigma, cfg.noise_frac,
                             cfg.center_seed, cfg.base_seed, 0, 0))
q = torch.empty(args.nq * cfg.d, dtype=torch.uint8, device="cuda")
check(lib().gann_generate_u8(q.data_ptr(), args.nq, cfg.d, cfg.clusters, cfg.sigma, cfg.noise_frac,
                             cfg.center_seed, cfg.query_seed, 0, 0))
idx = g.Index.from_device(base.data_ptr(), cfg.n, cfg.d, np.uint8, "l2", cfg.R)
idx.build(g.DiskannParams(cfg.R, cfg.L, cfg.alpha, max_batch=cfg.max_batch))
r = idx.search(q.cpu().numpy().reshape(args.nq, cfg.d), g.SearchParams(args.L, args.L, 0.0), k_out=10)
nv = r.n_visited.astype(np.float64)
dc = r.dist_comps.astype(np.float64)
pct = lambda a: " ".join(f"p{p}={np.percentile(a, p):.0f}" for p in (0, 1, 10, 50, 90, 99, 100))
print(f"|V|: mean {nv.mean():.1f} cv {nv.std() / nv.mean():.3f}  {pct(nv)}")
print(f"evals: mean {dc.mean():.1f} cv {dc.std() / dc.mean():.3f}  {pct(dc)}")

# cheap predictors of a query's cost at L: a short search's |V|, evaluations and best distance
for Lp in (10, 20, 40):
    p = idx.search(q.cpu().numpy().reshape(args.nq, cfg.d), g.SearchParams(Lp, Lp, 0.0), k_out=10)
    for name, x in (("|V|", p.n_visited.astype(np.float64)), ("evals", p.dist_comps.astype(np.float64)),
                    ("d1", p.dists[:, 0].astype(np.float64)), ("d10", p.dists[:, 9].astype(np.float64))):
        c = np.corrcoef(x, nv)[0, 1]
        # share of the 10% most expensive queries found among the predictor's top 20%
        top = nv >= np.percentile(nv, 90)
        pick = x >= np.percentile(x, 80)
        print(f"L={Lp} {name:6s} corr with |V|@{args.L}: {c:+.3f}  top-10% recall in predictor top-20%: "
              f"{(top & pick).sum() / top.sum():.2f}")
