"""Workloads for the checked library (tests/test_gpu_checked.py).

  GANN_LIB=libgann_checked.so python tools/checked_case.py small
  GANN_LIB=libgann_checked.so python tools/checked_case.py c0

Prints one JSON line: the checksums of the results and the checked build's
report (gann_debug_check: the largest source line of a failed bounds check).

Every kernel family of the path runs at least once: the start vertex, the
batch searches and binned / chunked / tensor-core prunes of a build, the
back-edge count / scatter / merge / re-prune, the query search in its three
visited modes, ground truth, explicit alpha_prune and group_by_key. Only
numpy and the package (ctypes) are imported."""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_04359_b200 as g  # noqa: E402
from paper_2305_04359_b200 import datagen  # noqa: E402


OUT = {}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()[:16]


def small():
    rng = np.random.default_rng(5)
    n, d = 3000, 32
    centers = rng.integers(0, 256, (10, d))
    data = np.clip(np.rint(centers[rng.integers(0, 10, n)] + rng.normal(0, 20, (n, d))), 0, 255).astype(np.uint8)
    qs = data[:64].copy()
    idx = g.build_diskann(data, "l2", g.DiskannParams(24, 48, 1.2, max_batch=300))
    OUT["small_graph"] = sha(idx.export_graph()[0])
    for mode in ("fast", "ref", "exact"):
        OUT["small_" + mode] = sha(idx.search(qs, g.SearchParams(48, 48, 0.0), visited_mode=mode, vcap=200).ids)
    OUT["small_eps"] = sha(idx.search(qs, g.SearchParams(32, 10, 0.25)).ids)
    OUT["small_gt"] = sha(idx.groundtruth(qs, 10)[0])
    # explicit prunes: a short list (tensor-core bins) and a hub list (chunked kernel)
    ids = [rng.choice(n, 100, replace=False).astype(np.uint32), rng.choice(n, 900, replace=False).astype(np.uint32)]
    dl = [((data[i].astype(np.int64) - data[0]) ** 2).sum(1).astype(np.float32) for i in ids]
    OUT["small_prune"] = sha(np.concatenate(idx.alpha_prune_many([0, 0], ids, dl, g.PruneParams(24, 1.2))))
    keys = rng.integers(0, 50, 5000).astype(np.uint32)
    gp = g.group_by_key(keys, np.arange(5000, dtype=np.uint32))
    order = np.argsort(gp.keys, kind="stable")  # group order is unspecified: canonical by key
    OUT["small_groups"] = sha(np.stack([gp.keys[order], gp.vals[order]]))
    # f32 rows: the warp prune and CUDA-core distances
    f = rng.normal(0, 1, (1500, 24)).astype(np.float32)
    fi = g.build_diskann(f, "l2", g.DiskannParams(16, 32, 1.2))
    OUT["small_f32"] = sha(fi.search(f[:32], g.SearchParams(32, 32, 0.0)).ids)


def c0():
    cfg = datagen.CONFIGS["c0"]
    data = datagen.host_base(cfg)
    qs = datagen.host_queries(cfg, 500)
    idx = g.build_diskann(data, "l2", g.DiskannParams(cfg.R, cfg.L, cfg.alpha, max_batch=cfg.max_batch))
    OUT["c0_graph"] = sha(idx.export_graph()[0])
    OUT["c0_L128"] = sha(idx.search(qs, g.SearchParams(128, 128, 0.0), vcap=400).ids)
    OUT["c0_L200_ref"] = sha(idx.search(qs, g.SearchParams(200, 200, 0.0), visited_mode="ref").ids)
    OUT["c0_L832"] = sha(idx.search(qs, g.SearchParams(832, 832, 0.0)).ids)


if __name__ == "__main__":
    import ctypes as C

    from paper_2305_04359_b200._lib import LIB_PATH, check, lib
    {"small": small, "c0": c0}[sys.argv[1]]()
    line, checked = C.c_uint32(), C.c_int()
    check(lib().gann_debug_check(0, C.byref(line), C.byref(checked)))
    print(json.dumps({"lib": LIB_PATH.name, "checked_build": checked.value, "failed_line": line.value, "out": OUT}))
