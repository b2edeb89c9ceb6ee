"""Build the config index on the GPU `--reps` times in one process and print
each build's wall time and phase split (the first build pays allocation).

  python tools/bench_build.py --n 10000000 --reps 2
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2305_04359_b200 as g  # noqa: E402
from paper_2305_04359_b200 import datagen  # noqa: E402
from paper_2305_04359_b200._lib import check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
cfg = datagen.CONFIGS[args.config].scaled(args.n)
torch.cuda.set_stream(torch.cuda.Stream())
tdt = {"u8": torch.uint8, "i8": torch.int8, "f32": torch.float32}[cfg.dtype]
base = torch.empty(cfg.n * cfg.d, dtype=tdt, device="cuda")
check(datagen.generate_device(lib(), cfg, base.data_ptr(), cfg.n, queries=False))
idx = g.Index.from_device(base.data_ptr(), cfg.n, cfg.d, cfg.np_dtype, cfg.metric, cfg.R)
sums = []
for r in range(args.reps):
    idx.reset_stats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    idx.build(g.DiskannParams(cfg.R, cfg.L, cfg.alpha, max_batch=cfg.max_batch))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    adj, deg, start = idx.export_graph()
    sums.append(int((adj.astype(np.uint64) * (np.arange(adj.size, dtype=np.uint64).reshape(adj.shape) % 7919 + 1)).sum()))
    ph = {k: round(v, 1) for k, v in idx.stats()["build_ms"].items()}
    print(f"build {r}: {dt:.3f} s  {cfg.n / dt / 1e6:.3f} M pts/s  phases {ph}  checksum {sums[-1]}", flush=True)
assert len(set(sums)) == 1, "builds differ"
