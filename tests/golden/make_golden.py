"""Generate the golden fixtures under tests/golden/ from the reference itself.

Runs the reference's own sources (compiled by oracle/Makefile into
oracle/_ref/libgraphann_ref.so) on small seeded inputs and stores inputs and
outputs. Regenerate with:  python tests/golden/make_golden.py
(needs /root/reference to build oracle/_ref; the fixtures are committed).
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from helpers import mixture  # noqa: E402
from oracle.oracle import Oracle, build  # noqa: E402

SETTINGS = [(10, 10, 0.0), (16, 10, 0.1), (32, 32, 0.0), (8, 4, 0.25), (2, 1, 0.0)]


def main():
    build(with_ref=True)
    ref = Oracle("ref")
    # --- search over the reference's own graph ---------------------------------------
    data, qs = mixture(101, 2000, 16, clusters=10, nq=64)
    adj, start = ref.build(data, 16, 32, 1.2, workers=2)
    out = dict(data=data, queries=qs, adj=adj, start=np.uint32(start))
    for i, (L, k, eps) in enumerate(SETTINGS):
        r = ref.beam_search(adj, start, data, qs, L, k, eps, visited_mode=1, vcap=4 * L + 16, workers=2)
        for key, v in r.items():
            out[f"s{i}_{key}"] = v
    np.savez_compressed(HERE / "search_u8.npz", **out, settings=np.array(SETTINGS, np.float64))
    # --- alpha_prune on the reference's visited lists -----------------------------------
    vis = ref.beam_search(adj, start, data, data[:40], 32, 32, vcap=160, workers=2)
    pr = {}
    for ci, (R, alpha, rule) in enumerate([(8, 1.2, "scale_candidate"), (8, 1.0, "scale_candidate"),
                                          (16, 0.9, "scale_selected"), (4, 2.0, "scale_candidate")]):
        outs, lens = [], []
        for i in range(40):
            nv = int(vis["n_visited"][i])
            kept, _ = ref.alpha_prune(i, vis["visited_ids"][i, :nv], vis["visited_dists"][i, :nv], data, R,
                                      alpha, rule)
            row = np.full(R, 0xFFFFFFFF, np.uint32)
            row[: len(kept)] = kept
            outs.append(row)
        pr[f"c{ci}_out"] = np.stack(outs)
        pr[f"c{ci}_params"] = np.array([R, alpha, 0 if rule == "scale_candidate" else 1], np.float64)
    np.savez_compressed(HERE / "prune_u8.npz", data=data, vis_ids=vis["visited_ids"], vis_dists=vis["visited_dists"],
                        n_visited=vis["n_visited"], **pr)
    # --- semisort ----------------------------------------------------------------------
    rng = np.random.default_rng(7)
    keys = rng.integers(0, 200, 3000).astype(np.uint32)
    vals = rng.integers(0, 2**32, 3000, dtype=np.uint64).astype(np.uint32)
    ok, ov, off = ref.group_by_key(keys, vals)
    np.savez_compressed(HERE / "semisort.npz", keys=keys, vals=vals, out_keys=ok, out_vals=ov, offsets=off)
    # --- builds -----------------------------------------------------------------------
    bdata = mixture(102, 1500, 16, clusters=8)
    g0, s0 = ref.build(bdata, 12, 24, 1.2, workers=2)
    g1, s1 = ref.build(bdata, 12, 24, 1.2, cap=50, workers=2)
    idata = mixture(103, 1200, 12, clusters=6, dtype=np.int8)
    g2, s2 = ref.build(idata, 10, 20, 0.9, rule="scale_selected", metric="ip", workers=2)
    fdata = mixture(104, 800, 8, clusters=5, dtype=np.float32)
    g3, s3 = ref.build(fdata, 10, 20, 1.0, metric="ip", workers=2)
    np.savez_compressed(HERE / "build.npz", u8=bdata, u8_uncapped=g0, u8_uncapped_start=np.uint32(s0),
                        u8_cap50=g1, u8_cap50_start=np.uint32(s1), i8=idata, i8_ip_sel=g2,
                        i8_ip_sel_start=np.uint32(s2), f32=fdata, f32_ip=g3, f32_ip_start=np.uint32(s3))
    # --- ground truth, start, schedule -----------------------------------------------------
    gi, gd = ref.groundtruth(data, qs, 16, workers=2)
    np.savez_compressed(HERE / "groundtruth.npz", ids=gi, dists=gd)
    sched = {
        "batch_ranges": {f"{n}/{cap}": ref.batch_ranges(n, cap) for n, cap in
                         [(1, 0), (2, 0), (3, 0), (8, 0), (10, 0), (1000, 0), (100000, 0), (100000, 2000), (5000, 97)]},
        "shuffled_order_100_42_33": ref.shuffled_order(100, 42, 33).tolist(),
        "shuffled_order_1000_insert_seed": ref.shuffled_order(1000, 16503569613174706033, 5).tolist(),
        "choose_start": {"u8": ref.choose_start(bdata), "i8_ip": ref.choose_start(idata, "ip"),
                         "f32_ip": ref.choose_start(fdata, "ip")},
    }
    (HERE / "schedule.json").write_text(json.dumps(sched))
    for f in sorted(HERE.glob("*")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
