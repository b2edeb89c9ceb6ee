"""Workloads for compute-sanitizer runs (tests/test_gpu_sanitizer.py).

  compute-sanitizer --tool racecheck python tools/sanitize_case.py small
  compute-sanitizer --tool memcheck  python tools/sanitize_case.py c0

Every kernel family of the path runs at least once: the start vertex, the
batch searches and binned / chunked / tensor-core prunes of a build, the
back-edge count / scatter / merge / re-prune, the query search in its three
visited modes, ground truth, explicit alpha_prune and group_by_key. Only
numpy and the package (ctypes) are imported: no torch under the sanitizer."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_04359_b200 as g  # noqa: E402
from paper_2305_04359_b200 import datagen  # noqa: E402


def small():
    rng = np.random.default_rng(5)
    n, d = 3000, 32
    centers = rng.integers(0, 256, (10, d))
    data = np.clip(np.rint(centers[rng.integers(0, 10, n)] + rng.normal(0, 20, (n, d))), 0, 255).astype(np.uint8)
    qs = data[:64].copy()
    idx = g.build_diskann(data, "l2", g.DiskannParams(24, 48, 1.2, max_batch=300))
    for mode in ("fast", "ref", "exact"):
        idx.search(qs, g.SearchParams(48, 48, 0.0), visited_mode=mode, vcap=200)
    idx.search(qs, g.SearchParams(32, 10, 0.25))
    idx.groundtruth(qs, 10)
    # explicit prunes: a short list (tensor-core bins) and a hub list (chunked kernel)
    ids = [rng.choice(n, 100, replace=False).astype(np.uint32), rng.choice(n, 900, replace=False).astype(np.uint32)]
    dl = [((data[i].astype(np.int64) - data[0]) ** 2).sum(1).astype(np.float32) for i in ids]
    idx.alpha_prune_many([0, 0], ids, dl, g.PruneParams(24, 1.2))
    keys = rng.integers(0, 50, 5000).astype(np.uint32)
    g.group_by_key(keys, np.arange(5000, dtype=np.uint32))
    # f32 rows: the warp prune and CUDA-core distances
    f = rng.normal(0, 1, (1500, 24)).astype(np.float32)
    fi = g.build_diskann(f, "l2", g.DiskannParams(16, 32, 1.2))
    fi.search(f[:32], g.SearchParams(32, 32, 0.0))


def c0():
    cfg = datagen.CONFIGS["c0"]
    data = datagen.host_base(cfg)
    qs = datagen.host_queries(cfg, 500)
    idx = g.build_diskann(data, "l2", g.DiskannParams(cfg.R, cfg.L, cfg.alpha, max_batch=cfg.max_batch))
    idx.search(qs, g.SearchParams(128, 128, 0.0), vcap=400)
    idx.search(qs, g.SearchParams(200, 200, 0.0), visited_mode="ref")


if __name__ == "__main__":
    {"small": small, "c0": c0}[sys.argv[1]]()
    print("sanitize case done")
