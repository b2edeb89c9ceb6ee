"""Build an index on the GPU and run the search kernel a few times (for ncu).

  python tools/profile_search.py --n 2000000 --L 128 --reps 3
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import os  # noqa: E402

os.environ.setdefault("GANN_SEARCH_DIAG", "1")  # per-query diagnostic counters (general kernel)
import paper_2305_04359_b200 as g  # noqa: E402
from paper_2305_04359_b200 import datagen  # noqa: E402
from paper_2305_04359_b200._lib import check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--nq", type=int, default=10_000)
ap.add_argument("--L", type=int, default=128)
ap.add_argument("--Ls", default="", help="comma list: search several beams on one build")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
cfg = datagen.CONFIGS[args.config].scaled(args.n)
torch.cuda.set_stream(torch.cuda.Stream())
base = torch.empty(cfg.n * cfg.d, dtype=torch.uint8, device="cuda")
check(lib().gann_generate_u8(base.data_ptr(), cfg.n, cfg.d, cfg.clusters, cfg.sigma, cfg.noise_frac,
                             cfg.center_seed, cfg.base_seed, 0, 0))
q = torch.empty(args.nq * cfg.d, dtype=torch.uint8, device="cuda")
check(lib().gann_generate_u8(q.data_ptr(), args.nq, cfg.d, cfg.clusters, cfg.sigma, cfg.noise_frac,
                             cfg.center_seed, cfg.query_seed, 0, 0))
idx = g.Index.from_device(base.data_ptr(), cfg.n, cfg.d, np.uint8, "l2", cfg.R)
t0 = time.time()
idx.build(g.DiskannParams(cfg.R, cfg.L, cfg.alpha, max_batch=cfg.max_batch))
torch.cuda.synchronize()
print(f"build {time.time() - t0:.2f}s", idx.stats()["build_ms"], flush=True)
idx.stage_queries(q.data_ptr(), args.nq)
ids = torch.empty(args.nq * 10, dtype=torch.int32, device="cuda")
ds = torch.empty(args.nq * 10, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
torch.cuda.synchronize()
idx.reset_stats()
torch.cuda.profiler.start()  # ncu --profile-from-start off captures only these launches
import os  # noqa: E402
Ls = [int(x) for x in args.Ls.split(",")] if args.Ls else [args.L]
for L in Ls:
    for hl in ([int(x) for x in os.environ.get("HLOGS", "").split(",") if x] or [0]):
        if hl:
            os.environ["GANN_HASH_LOG2"] = str(hl)
        best = 1e9
        idx.reset_stats()
        for r in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if os.environ.get("MODE", "fast") == "fast":
                idx.search_staged(g.SearchParams(L, L, 0.0), 10, ids.data_ptr(), ds.data_ptr(), s.cuda_stream)
            else:
                idx.search_device(q.data_ptr(), args.nq, g.SearchParams(L, L, 0.0), 10, ids.data_ptr(), ds.data_ptr(),
                                  stream=s.cuda_stream, visited_mode=os.environ["MODE"])
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        st = idx.stats()
        nqq = max(1, st["queries"])
        print(f"search L={L} H=2^{hl or 'default'}: {best:.3f} ms  evals/q {st['evaluations'] / nqq:.1f}  "
              f"exp/q {st['expansions'] / nqq:.1f}  survivors/q {st['survivors'] / nqq:.1f}  "
              f"moved/q {st['moved'] / nqq:.1f}  dups/q {st['duplicates'] / nqq:.1f}", flush=True)
torch.cuda.profiler.stop()
st = idx.stats()
print("stats", {k: st[k] for k in ("queries", "expansions", "evaluations", "filter_drops", "adj_entries", "merges", "survivors", "moved")})
