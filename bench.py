#!/usr/bin/env python
"""Benchmark: batched beam-search QPS over a Vamana graph built from BASELINE
config 1 (10M x 128 u8, R64 L128 alpha 1.2), at the smallest beam of the
BASELINE sweep (10..200) reaching recall@10 0.95, else at L=200; plus the
QPS / recall curve over every beam of the sweep and past it, the build's
points/s and roofline, the search kernel's HBM roofline, the end-to-end QPS
through the C ABI with host buffers, and the reference's CPU search timed
beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--n N]
  python bench.py --impl reference ...     # the reference's own CPU path

A step is one search launch over one batch of 10,000 queries per GPU (the
config's query set); the index (1.28 GB vectors + 2.56 GB graph) is larger
than L2, so no flush is needed between steps (smaller indexes are flushed,
and then launch serially). Steps alternate over two streams, so one batch's
tail (its last, longest queries) overlaps the next batch's start, as a
serving loop would; every step still searches its whole batch. e2e runs the
same loop through gann_search_async with pinned host buffers (H2D + search +
D2H per step); the blocking gann_search is reported beside it.
Multi-GPU: one process per GPU; one vertex-partitioned build over all GPUs
(NCCL all-to-all-v of reverse pairs), the rows all-gathered into a replica
per rank (checksum all-gather verifies them); each rank searches its own
10k-query shard — no data-path collective ("scaling": "weak"). Timing: CUDA
events on the launching streams, barrier + synchronize on both sides, max
over ranks.

The reference arm (--impl reference) never imports the package: it
regenerates the config's points on the host (datagen's numpy restatement,
bit-identical to the device generator), builds the graph with graphann's own
build loop (oracle/_ref: the reference's sources), computes graphann's ground
truth, and times graphann's beam_search on all host threads. Both arms print
the same `config`, the graph's and the headline ids' SHA-256 (`parity`), and a
QPS / recall curve (`qps_curve`).
"""
from __future__ import annotations

import argparse
import ctypes
import hashlib
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# BASELINE.json: "beam L swept 10..200"; --L-max widens it
L_CANDIDATES = [10, 12, 14, 16, 20, 24, 28, 32, 40, 48, 56, 64, 80, 96, 128, 160, 200, 256, 320, 400, 512]
# beams tried past the sweep while the recall target is not reached (both arms;
# ours stops at the kernel's on-chip beam limit, gann_search_max_beam)
L_EXTEND = [256, 320, 400, 512, 640, 800, 1024, 1280, 1600, 2048, 2560, 3200, 4096, 5120, 6400, 8192]
GT_DEPTH = 16
CFG_INDEX = {"c0": 0, "c1": 1, "c2": 2, "c3": 3, "c4": 4}  # BASELINE.json configs[i]
B200_L2_BYTES = 126 * 2**20
METRIC = ("search QPS at recall@10 0.95 (Alg.1 beam {L,L,0}, top-10): the smallest beam reaching it, searched "
          "over the BASELINE sweep 10..200, continued past 200 and bisected to a multiple of 32 (config carries L and "
          "its recall; qps_curve every beam tried)")


def load_module(name, rel):
    spec = importlib.util.spec_from_file_location(name, ROOT / rel)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


# datagen / evalutil are plain numpy: load them without importing the package
# (which loads libgann_b200.so) so the reference arm never touches our library.
datagen = load_module("gann_datagen", "paper_2305_04359_b200/datagen.py")
evalutil = load_module("gann_evalutil", "paper_2305_04359_b200/evalutil.py")
distutil = load_module("gann_distutil", "paper_2305_04359_b200/distutil.py")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1")
    # (--points / --queries: torchrun's own argument parser claims --n / --nq prefixes)
    ap.add_argument("--n", "--points", dest="n", type=int, default=0, help="override the config's n (debug)")
    ap.add_argument("--nq", "--queries", dest="nq", type=int, default=0, help="queries per GPU (default: the config's)")
    ap.add_argument("--target-recall", type=float, default=0.95)
    ap.add_argument("--L", type=int, default=0, help="force the search beam")
    ap.add_argument("--L-max", type=int, default=200, help="largest beam of the sweep (BASELINE: 10..200)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline sample length")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extend", action="store_true",
                    help="do not search past the sweep for the beam that reaches the recall target")
    ap.add_argument("--ref-build", default="full", choices=["full", "prefix"],
                    help="reference arm: build the config's whole graph with graphann (default) or only a "
                         "--ref-n prefix (quick checks; then the search runs over that prefix's graph)")
    ap.add_argument("--ref-n", type=int, default=100_000, help="reference arm: points of a prefix build")
    ap.add_argument("--streams", type=int, default=2,
                    help="timed steps alternate over this many streams, so one step's tail overlaps the next "
                         "step's start (1 = serial launches; forced to 1 when steps flush L2)")
    ap.add_argument("--no-build-roofline", action="store_true",
                    help="skip the untimed exact-count rebuild behind build.roofline")
    ap.add_argument("--search-on", default="auto", choices=["auto", "replica", "partitions"],
                    help="N>1 after the partitioned build: gather a full graph replica per rank (when it fits) "
                         "or search the partitions in place (peer rows over NVLink)")
    ap.add_argument("--replicated-build", action="store_true",
                    help="N>1: every rank builds the whole graph (default: one vertex-partitioned build)")
    return ap.parse_args()


def workload(args):
    cfg = datagen.CONFIGS[args.config]
    if args.n:
        cfg = cfg.scaled(args.n)
    return cfg, (args.nq or cfg.n_queries)


def sweep_beams(args):
    return [args.L] if args.L else [x for x in L_CANDIDATES if x <= args.L_max]


def choose_beam(args, curve, eval_L, max_beam=1 << 30):
    """The headline beam, by one rule in both arms (each on its own recall):
    the smallest beam of the sweep reaching the target; else the L_EXTEND
    beams past the sweep until one reaches it, then bisection between the
    last miss and that hit on multiples of 32. eval_L(L) -> (recall, extra)
    runs one beam. Returns (L, reached, extension points). If no beam up to
    max_beam reaches the target, the beam with the highest recall tried."""
    if args.L:
        return args.L, None, []
    for c in curve:
        if c["recall@10"] >= args.target_recall:
            return c["L"], True, []
    ext = []
    if args.no_extend:
        return curve[-1]["L"], False, ext

    def run(L):
        rec, extra = eval_L(L)
        ext.append(dict({"L": L, "recall@10": round(rec, 5)}, **extra))
        return rec

    lo, hi = curve[-1]["L"], None
    for L in [x for x in L_EXTEND if x > lo]:
        if L > max_beam:
            break
        if run(L) >= args.target_recall:
            hi = L
            break
        lo = L
    if hi is None:
        best = max([(c["recall@10"], c["L"]) for c in curve] + [(e["recall@10"], e["L"]) for e in ext])
        return best[1], False, ext
    while hi - lo > 32:
        mid = max(lo + 32, (lo + hi) // 64 * 32)
        if run(mid) >= args.target_recall:
            hi = mid
        else:
            lo = mid
    return hi, True, sorted(ext, key=lambda e: e["L"])


def config_obj(args, cfg, nq, L, recall):
    """The workload both arms print, key for key."""
    index_bytes = cfg.n * (cfg.d * cfg.elem_bytes + 4 * cfg.R)
    return {
        "workload": f"BASELINE configs[{CFG_INDEX.get(args.config, '?')}]: {cfg.name}",
        "n": cfg.n, "d": cfg.d, "dtype": cfg.dtype, "metric": cfg.metric, "R": cfg.R, "L_build": cfg.L,
        "alpha": cfg.alpha, "max_batch": cfg.max_batch, "queries_per_gpu": nq, "k": cfg.k,
        "L_search": L, "recall@10": round(recall, 5), "target_recall": args.target_recall,
        "target_reached": recall >= args.target_recall,
        "graph": "built from the config's points by each arm (ours: gann_build on the GPU; reference: graphann's "
                 "build loop on the host); parity.graph_sha256 compares them",
        "l2": ("flushed between steps" if index_bytes < 2 * B200_L2_BYTES
               else f"inputs larger than L2 ({index_bytes / 1e9:.2f} GB index)"),
    }


def sha16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()[:16]


def build_bytes(st: dict, n: int, row_bytes: int, R: int):
    """Algorithmic bytes of a whole build: per inserted point j
    B_search(j) + |V_j| d s (prune rows) + 4R (its row written), per batch
    16 E_b (pairs written + read) + per target 4(1+deg) read + 4(1+deg') written
    + |M_t| d s when the merged list is re-pruned. `st` must come from a build
    whose searches counted distinct evaluations (EXACT visited mode): then
    st["evaluations"] = sum_j U_j. |V_j| = the expansions; the re-prune lists'
    candidates = all prune candidates - the insert lists'."""
    U, V = st["evaluations"], st["expansions"]
    reprune_cands = max(0, st["prune_candidates"] - V)
    search = U * row_bytes + 4.0 * V * (1 + R) + n * row_bytes
    prune = V * row_bytes + 4.0 * R * n
    back = 16.0 * st["back_pairs"] + 8.0 * (1 + R) * st["back_groups"] + reprune_cands * row_bytes
    return {"search": search, "prune": prune, "back_edges": back, "total": search + prune + back}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = Path(f"/tmp/gann_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", os.environ.get("GANN_CLOCK_MS", "50")],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None
        time.sleep(0.2)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        self.proc.wait()
        rows = [l.split(", ") for l in self.path.read_text().strip().splitlines() if l.count(",") >= 7]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        sm = []
        smax = None
        for r in rows:
            try:
                sm.append(float(r[0]))
                smax = float(r[1])
            except ValueError:
                continue
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def search_bytes(stats: dict, row_bytes: int, nq: int, k: int) -> float:
    """Algorithmic bytes of a search launch:
    B = sum_q [U_q*d*s + sum_{v in V_q} 4*(1 + deg v) + d*s + 8k], with the
    distinct-evaluation count U from an EXACT visited-mode run of the same
    queries (stats["evaluations"] there), |V| and sum deg from the same run."""
    # the fast-mode kernel keeps no adjacency counter (diagnostics off): count
    # the full R-wide row it reads per expansion instead
    adj = stats["adj_entries"] or stats["expansions"] * stats.get("R", 64)
    return (stats["evaluations"] * row_bytes + 4.0 * (stats["expansions"] + adj)
            + nq * row_bytes + 8.0 * k * nq)


def gathered_obj(sstats: dict, steps: int, row_bytes: int, nq: int, k: int, R: int, launch_s: float, peak: float,
                 traffic):
    """What the fast kernel actually moves per launch: every row it scores
    (re-evaluations of ids its visited table dropped included) plus the
    adjacency rows, against the same HBM peak; and the ncu DRAM traffic of the
    same launch as a bandwidth. The roofline's `achieved` counts distinct
    evaluations only, so it is the conservative one."""
    per = search_bytes(dict(sstats, evaluations=sstats["evaluations"] / steps,
                            expansions=sstats["expansions"] / steps, adj_entries=0, R=R), row_bytes, nq, k)
    rate = per / launch_s / 1e9
    out = {"basis": "scored rows x row bytes + R-wide adjacency rows per expansion (the fast visited table's "
                    "re-evaluations included; many are L2 hits)",
           "bytes_per_launch": round(per), "rate": round(rate, 1), "unit": "GB/s", "frac": round(rate / peak, 4)}
    if traffic:
        out["dram_traffic_rate"] = round(traffic / launch_s / 1e9, 1)
        out["dram_traffic_frac"] = round(traffic / launch_s / 1e9 / peak, 4)
    return out


def traffic_from_profile(workload: str, L: int):
    """dram bytes (read + write) of one timed launch from an ncu --set full
    capture of the same workload and beam (profiles/traffic.json), else None."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        d = json.loads(p.read_text()).get(workload, {})
        if d.get("L") == L:
            return d.get("search_kernel_bytes")
    return None


# ---------------------------------------------------------------------------------
def setup(args):
    """Data in HBM, the GPU build (timed once), ground truth and the beam L
    that reaches the recall target. Shared by both arms."""
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    # GANN_BENCH_BACKEND=gloo: a check of the N>1 logic on a one-GPU box (ranks
    # share the device, collectives staged through the host); never a number
    backend = os.environ.get("GANN_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    # a dedicated stream: torch's legacy default stream has handle 0, which the C
    # ABI reads as "the index's own stream"
    torch.cuda.set_stream(torch.cuda.Stream())
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_2305_04359_b200 as g
    from paper_2305_04359_b200._lib import check, lib

    cfg, nq = workload(args)
    n, d, k = cfg.n, cfg.d, cfg.k
    dev = local

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allreduce(x, op="max"):
        return distutil.reduce_scalar(x, op, dist if world > 1 else None, "cuda" if backend == "nccl" else "cpu")

    # ---- data: generated straight into HBM ------------------------------------------
    # (N>1, partitioned build of rows that need no padding: straight into the
    # partition index's own buffer — a 1B-point set fits once, not twice)
    tdt = {"u8": torch.uint8, "i8": torch.int8, "f32": torch.float32}[cfg.dtype]
    in_place = world > 1 and not args.replicated_build and (d * cfg.elem_bytes) % 16 == 0
    base = None if in_place else torch.empty(n * d, dtype=tdt, device="cuda")
    if base is not None:
        check(datagen.generate_device(lib(), cfg, base.data_ptr(), n, queries=False, device=dev))
    qdev = torch.empty(nq * d, dtype=tdt, device="cuda")
    row0, _ = distutil.query_rows(rank, nq)  # each rank searches its own query shard
    check(datagen.generate_device(lib(), cfg, qdev.data_ptr(), nq, queries=True, row0=row0, device=dev))
    # ---- build (timed once) ---------------------------------------------------------------
    params = g.DiskannParams(cfg.R, cfg.L, cfg.alpha, seed=42, max_batch=cfg.max_batch)
    build_mode, search_on, build_extra, pidx, idx = "single-gpu", "replica", {}, None, None
    if world > 1 and not args.replicated_build:
        # one vertex-partitioned build over the N GPUs: the C++ batch loop
        # (gann_part_build) with the library's NCCL transport; peer rows over
        # NVLink (CUDA IPC). The batch cap is the config's, shrunk to what the
        # free device memory holds (0.2-0.5% of n at 1B).
        from paper_2305_04359_b200.partition import DistExchange, NcclExchange, PartitionedIndex
        pidx = PartitionedIndex(base.data_ptr() if base is not None else 0, cfg.metric, cfg.R, dist, device=dev,
                                shape=(n, d), dtype=cfg.np_dtype)
        if base is None:
            pts_ptr, _ = pidx.device_points()
            check(datagen.generate_device(lib(), cfg, pts_ptr, n, queries=False, device=dev))
            base = _tensor_from_ptr(pts_ptr, n * d * cfg.elem_bytes).view(tdt)  # a view of the index's points
        if pidx.peers_ok:
            free_b, _ = torch.cuda.mem_get_info(dev)
            # the full replica (points are already resident: graph rows only)
            # is gathered for the search when it fits; else the search reads
            # the partitions in place
            replica_b = n * cfg.R * 4 + n * d * cfg.elem_bytes
            search_on = args.search_on if args.search_on != "auto" else (
                "replica" if replica_b < 0.4 * free_b else "partitions")
            mem_cap = pidx.batch_cap(cfg.L, int(0.8 * free_b))
            cap = int(allreduce(min(cfg.max_batch or n, mem_cap), "min"))
            params = g.DiskannParams(cfg.R, cfg.L, cfg.alpha, seed=42, max_batch=cap)
            xch = NcclExchange(dist, dev) if backend == "nccl" else DistExchange(dist, dev)
            barrier()
            t0 = time.perf_counter()
            info = pidx.build_native(params, xch)
            torch.cuda.synchronize()
            build_s = allreduce(time.perf_counter() - t0)
            if backend == "nccl":
                xch.close()
            bstats = pidx.stats()  # this rank's share of the build
            build_mode = (f"vertex-partitioned over {world} GPUs (gann_part_build, "
                          + ("NCCL send/recv exchange)" if backend == "nccl" else f"{backend} exchange: logic check)"))
            build_extra = {"max_batch_used": cap, "max_batch_memory_cap": mem_cap, "pairs_sent": info["pairs_sent"],
                           "search_on": search_on}
            if search_on == "replica":
                P = -(-n // world)
                rows = torch.full((P * cfg.R,), -1, dtype=torch.int32, device="cuda")
                rows[: pidx.rows * cfg.R] = pidx.device_rows()
                full = torch.empty((world * P * cfg.R,), dtype=torch.int32, device="cuda")
                if backend == "nccl":
                    dist.all_gather_into_tensor(full, rows)
                else:  # host-staged
                    parts = [torch.empty(P * cfg.R, dtype=torch.int32) for _ in range(world)]
                    dist.all_gather(parts, rows.cpu())
                    full.copy_(torch.cat(parts).cuda())
                idx = g.Index.from_device(base.data_ptr(), n, d, cfg.np_dtype, cfg.metric, cfg.R, dev)
                check(lib().gann_import_graph_device(idx._h, ctypes.c_void_p(full.data_ptr()), pidx.start()))
                del full, rows
                pidx.close()
                pidx = None
                if in_place:  # the view into the closed partition's points moves to the replica's
                    base = _tensor_from_ptr(idx.device_ptrs()[0], n * d * cfg.elem_bytes).view(tdt)
            else:
                idx = pidx.as_index()  # searches read every partition in place
        else:
            pidx.close()
            pidx = None
    if idx is None:
        idx = g.Index.from_device(base.data_ptr(), n, d, cfg.np_dtype, cfg.metric, cfg.R, dev)
        idx.reset_stats()
        # optional warm-up build (GANN_BENCH_WARM_BUILD=<points>); off by default:
        # measured no faster, and the timed build's re-prune then varied more
        nw = min(n, int(os.environ.get("GANN_BENCH_WARM_BUILD", 0)))
        if nw:
            widx = g.Index.from_device(base.data_ptr(), nw, d, cfg.np_dtype, cfg.metric, cfg.R, dev)
            widx.build(g.DiskannParams(cfg.R, cfg.L, cfg.alpha, seed=42, max_batch=int(nw * cfg.batch_cap_frac)))
            widx.close()
            del widx
        barrier()
        barrier()
        t0 = time.perf_counter()
        idx.build(params)
        torch.cuda.synchronize()
        build_s = allreduce(time.perf_counter() - t0)
        if world > 1:
            build_mode = "replicated: every rank builds the whole graph"
        bstats = idx.stats()
    idx.release_scratch()  # after the timed build: the search needs none of it
    adj_h, deg_h, start_h = idx.export_graph()  # host copy: the graph's checksum (and the CPU baseline)
    if search_on == "partitions":  # each rank holds its own rows: the checksum of the rank checksums
        shas = [None] * world
        dist.all_gather_object(shas, sha16(adj_h))
        graph_sha = hashlib.sha256("".join(shas).encode()).hexdigest()[:16]
        replicas_identical = None
        deg_mean = allreduce(float(deg_h.sum()), "sum") / n
    else:
        graph_sha = sha16(adj_h)
        replicas_identical = distutil.replicas_identical(int(graph_sha, 16), dist if world > 1 else None)
        deg_mean = float(deg_h.mean())

    # ---- ground truth (GPU brute force) -------------------------------------------
    if d * cfg.elem_bytes <= 256:
        gt_ids = torch.empty(nq * GT_DEPTH, dtype=torch.int32, device="cuda")
        gt_d = torch.empty(nq * GT_DEPTH, dtype=torch.float32, device="cuda")
        idx.groundtruth_device(qdev.data_ptr(), nq, GT_DEPTH, gt_ids.data_ptr(), gt_d.data_ptr())
        torch.cuda.synchronize()
        gt_ids_h = gt_ids.cpu().numpy().view(np.uint32).reshape(nq, GT_DEPTH)
        gt_d_h = gt_d.cpu().numpy().reshape(nq, GT_DEPTH)
    else:  # wide f32 rows (config 3): gann_groundtruth takes rows up to 256 B
        gt_ids_h, gt_d_h = groundtruth_wide_f32(torch, base.view(n, d), qdev.view(nq, d), cfg.metric, GT_DEPTH)
    idx.stage_queries(qdev.data_ptr(), nq)
    out_ids = torch.empty(nq * k, dtype=torch.int32, device="cuda")
    out_d = torch.empty(nq * k, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    # L2: flushed between steps when the index fits in it (serial launches then)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    index_bytes = n * (d * cfg.elem_bytes + 4 * cfg.R)
    flush = index_bytes < 2 * l2_bytes
    flush_buf = torch.empty(max(4 * l2_bytes, 1), dtype=torch.uint8, device="cuda") if flush else None
    nstreams = 1 if flush else max(1, args.streams)
    streams = [stream] + [torch.cuda.Stream().cuda_stream for _ in range(nstreams - 1)]
    souts = [(out_ids, out_d)] + [(torch.empty_like(out_ids), torch.empty_like(out_d)) for _ in range(nstreams - 1)]
    ext = [torch.cuda.ExternalStream(sp_) for sp_ in streams]

    def search_L(L):
        idx.search_staged(g.SearchParams(L, L, 0.0), k, out_ids.data_ptr(), out_d.data_ptr(), stream)

    def timed(sp, nt):
        """ms per launch of nt launches alternating over the streams (serial
        launches with L2 flushes when the index fits in L2), max over ranks."""
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nt)]
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        t0e.record(ext[0])
        for es in ext[1:]:
            es.wait_event(t0e)
        for i, (e0, e1) in enumerate(evs):
            j = i % nstreams
            if flush:
                flush_buf.fill_(1)
            e0.record(ext[j])
            idx.search_staged(sp, k, souts[j][0].data_ptr(), souts[j][1].data_ptr(), streams[j])
            e1.record(ext[j])
        for es in ext[1:]:
            ev = torch.cuda.Event()
            ev.record(es)
            ext[0].wait_event(ev)
        t1e.record(ext[0])
        torch.cuda.synchronize()
        barrier()
        spans = [e0.elapsed_time(e1) for e0, e1 in evs]
        total = sum(spans) if nstreams == 1 else t0e.elapsed_time(t1e)
        return allreduce(total) / nt, spans

    def recall_of(res, rows=None):
        ti, td = (gt_ids_h, gt_d_h) if rows is None else (gt_ids_h[:rows], gt_d_h[:rows])
        r = res if rows is None else res[:rows]
        return allreduce(float(evalutil.recall_at_k(ti, td, r, k).mean()), "mean")

    # ---- QPS / recall at every beam of the sweep, then the headline beam -------------------
    curve = []
    for L in sweep_beams(args):
        sp = g.SearchParams(L, L, 0.0)
        search_L(L)  # warm + results for the recall
        torch.cuda.synchronize()
        res = out_ids.cpu().numpy().view(np.uint32).reshape(nq, k)
        ms, _ = timed(sp, 4)
        curve.append({"L": L, "recall@10": round(recall_of(res), 5), "qps": round(world * nq / (ms / 1e3), 1),
                      "ms_per_launch": round(ms, 4)})
    max_beam = idx.max_beam()

    def eval_L(L):
        search_L(L)
        torch.cuda.synchronize()
        res = out_ids.cpu().numpy().view(np.uint32).reshape(nq, k)
        ms, _ = timed(g.SearchParams(L, L, 0.0), 2)
        return recall_of(res), {"qps": round(world * nq / (ms / 1e3), 1), "ms_per_launch": round(ms, 4)}

    chosen, target_reached, ext_curve = choose_beam(args, curve, eval_L, max_beam)
    recall = next(c["recall@10"] for c in curve + ext_curve if c["L"] == chosen)
    sp = g.SearchParams(chosen, chosen, 0.0)
    search_L(chosen)
    torch.cuda.synchronize()
    ids_sha = sha16(out_ids.cpu().numpy().view(np.uint32).reshape(nq, k))

    return dict(torch=torch, dist=dist, g=g, check=check, lib=lib, cfg=cfg, nq=nq, n=n, d=d, k=k, dev=dev,
                rank=rank, world=world, barrier=barrier, allreduce=allreduce, base=base, qdev=qdev, idx=idx,
                build_s=build_s, bstats=bstats, replicas_identical=replicas_identical, deg_mean=deg_mean,
                build_mode=build_mode, adj_h=adj_h, start_h=start_h, graph_sha=graph_sha, ids_sha=ids_sha,
                out_ids=out_ids, out_d=out_d, stream=stream, search_L=search_L, curve=curve, chosen=chosen,
                recall=recall, target_reached=target_reached, sp=sp, gt_ids_h=gt_ids_h, gt_d_h=gt_d_h,
                ext_curve=ext_curve, max_beam=max_beam, timed=timed, flush=flush,
                flush_buf=flush_buf, nstreams=nstreams, streams=streams, souts=souts, ext=ext,
                index_bytes=index_bytes, params=params, build_extra=build_extra, search_on=search_on)


def run_ours(args):
    S = setup(args)
    torch, dist, g, check, lib, cfg = S["torch"], S["dist"], S["g"], S["check"], S["lib"], S["cfg"]
    nq, n, d, k, dev, rank, world = S["nq"], S["n"], S["d"], S["k"], S["dev"], S["rank"], S["world"]
    barrier, allreduce, base, qdev, idx = S["barrier"], S["allreduce"], S["base"], S["qdev"], S["idx"]
    build_s, bstats, replicas_identical, deg_mean = S["build_s"], S["bstats"], S["replicas_identical"], S["deg_mean"]
    build_mode = S["build_mode"]
    out_ids, out_d, stream, search_L, curve = S["out_ids"], S["out_d"], S["stream"], S["search_L"], S["curve"]
    chosen, recall, target_reached, sp = S["chosen"], S["recall"], S["target_reached"], S["sp"]
    flush, flush_buf, nstreams, streams, souts, ext = (S["flush"], S["flush_buf"], S["nstreams"], S["streams"],
                                                       S["souts"], S["ext"])
    s_el = cfg.elem_bytes

    # ---- timed search steps --------------------------------------------------------
    for _ in range(args.warmup):
        search_L(chosen)
    idx.reset_stats()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(dev)
    sampler.start()
    barrier()
    if os.environ.get("GANN_PROFILE_RANGE"):
        torch.cuda.profiler.start()  # ncu --profile-from-start off: only the timed launches
    t_start.record(ext[0])
    for es in ext[1:]:
        es.wait_event(t_start)
    for i, (e0, e1) in enumerate(evs):
        j = i % nstreams
        if flush:
            flush_buf.fill_(1)
        e0.record(ext[j])
        idx.search_staged(sp, k, souts[j][0].data_ptr(), souts[j][1].data_ptr(), streams[j])
        e1.record(ext[j])
    for es in ext[1:]:
        ev = torch.cuda.Event()
        ev.record(es)
        ext[0].wait_event(ev)
    t_end.record(ext[0])
    torch.cuda.synchronize()
    barrier()
    if os.environ.get("GANN_PROFILE_RANGE"):
        torch.cuda.profiler.stop()
    clocks = sampler.stop()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]  # each launch on its stream (overlaps its neighbours)
    # serial launches: the sum of the launches' own spans (excludes the L2
    # flushes between them); pipelined: the elapsed time of all K launches
    total_ms = allreduce(sum(step_ms) if nstreams == 1 else t_start.elapsed_time(t_end))
    sstats = idx.stats()
    qps = world * nq * args.steps / (total_ms / 1e3)
    outs_agree = all(bool((o[0] == out_ids).all().item()) for o in souts[1:])
    # the algorithmic bytes of one launch: the same queries once more in EXACT mode
    idx.reset_stats()
    idx.search_device(qdev.data_ptr(), nq, sp, k, out_ids.data_ptr(), out_d.data_ptr(), stream=stream,
                      visited_mode="exact")
    torch.cuda.synchronize()
    xstats = idx.stats()
    per_launch_bytes = search_bytes(xstats, d * s_el, nq, k)
    # the same accounting at the last beam of the BASELINE sweep (context for the
    # headline: the kernel's fraction of the peak falls as the beam grows)
    sweep_end = None
    last = next((c for c in reversed(S["curve"]) if c["L"] != chosen), None) if S.get("curve") else None
    if last is not None:
        idx.reset_stats()
        tmp_ids, tmp_d = torch.empty_like(out_ids), torch.empty_like(out_d)  # (out_ids keeps the headline's ids)
        idx.search_device(qdev.data_ptr(), nq, g.SearchParams(last["L"], last["L"], 0.0), k, tmp_ids.data_ptr(),
                          tmp_d.data_ptr(), stream=stream, visited_mode="exact")
        torch.cuda.synchronize()
        lb = search_bytes(idx.stats(), d * s_el, nq, k)
        la = lb / (last["ms_per_launch"] / 1e3) / 1e9
        sweep_end = {"L": last["L"], "recall@10": last["recall@10"], "avg_launch_ms": last["ms_per_launch"],
                     "algorithmic_bytes_per_launch": round(lb), "achieved": round(la, 1),
                     "frac": round(la / peaks()[0], 4),
                     "kernel": "search_batch_kernel" if last["L"] >= 320 else "search_kernel"}
    # sustained time per launch: the K launches' elapsed time / K (with 2
    # streams a launch's own event span includes its overlap with neighbours)
    avg_launch_s = total_ms / args.steps / 1e3
    peak, peak_src = peaks()
    achieved = per_launch_bytes / avg_launch_s / 1e9

    # ---- end to end through the C ABI with host buffers -------------------------------------
    # every step: pinned host queries -> HBM, the search, ids + dists -> pinned
    # host buffers. gann_search_async enqueues a step on a stream with its own
    # scratch; steps alternate over the same streams as above. The blocking
    # gann_search is timed too (e2e.blocking).
    import ctypes as C
    qh = torch.empty((nq, d), dtype=qdev.dtype).pin_memory()
    qh.copy_(qdev.view(nq, d).cpu())
    hout = [(torch.empty((nq, k), dtype=torch.int32).pin_memory(), torch.empty((nq, k), dtype=torch.float32).pin_memory())
            for _ in range(nstreams)]
    scratch_b = idx.async_scratch_bytes(nq, k)
    scratch = [torch.empty(scratch_b, dtype=torch.uint8, device="cuda") for _ in range(nstreams)]
    L_ = lib()
    search_L(chosen)
    torch.cuda.synchronize()

    def e2e_async(i):
        j = i % nstreams
        idx.search_async(qh.data_ptr(), nq, sp, k, hout[j][0].data_ptr(), hout[j][1].data_ptr(),
                         scratch[j].data_ptr(), scratch_b, streams[j])

    for i in range(args.warmup):
        e2e_async(i)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        e2e_async(i)
    torch.cuda.synchronize()
    barrier()
    e2e_s = allreduce(time.perf_counter() - t0)
    ref_ids = out_ids.cpu().numpy().view(np.uint32).reshape(nq, k)
    e2e_match = all(bool((h[0].numpy().view(np.uint32) == ref_ids).all()) for h in hout)

    ih = hout[0][0]

    def e2e_blocking():
        check(L_.gann_search(idx.handle, C.c_void_p(qh.data_ptr()), nq, k, chosen, chosen, 0.0, 0, None,
                             C.c_void_p(ih.data_ptr()), C.c_void_p(hout[0][1].data_ptr()), None, None, None, None, 0))

    for _ in range(args.warmup):
        e2e_blocking()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_blocking()
    barrier()
    e2e_block_s = allreduce(time.perf_counter() - t0)
    e2e_match = e2e_match and bool((ih.numpy().view(np.uint32) == ref_ids).all())

    # ---- secondary sweep: the reference eval semantics {L, 10, eps} ----------
    secondary = []
    gt_ids_h, gt_d_h = S["gt_ids_h"], S["gt_d_h"]
    for eps in (0.0, 0.1, 0.25):
        for L in [x for x in (16, 32, 64, 128, 200) if x <= args.L_max]:
            spx = g.SearchParams(L, k, eps)
            idx.search_staged(spx, k, out_ids.data_ptr(), out_d.data_ptr(), stream)
            torch.cuda.synchronize()
            res = out_ids.cpu().numpy().view(np.uint32).reshape(nq, k)
            rec = float(evalutil.recall_at_k(gt_ids_h, gt_d_h, res, k).mean())
            ms, _ = S["timed"](spx, 3)
            secondary.append({"L": L, "k_gate": k, "eps": eps, "recall@10": round(allreduce(rec, "mean"), 5),
                              "qps": round(world * nq / (ms / 1e3), 1)})
    search_L(chosen)  # out_ids back to the headline search (the CPU baseline compares against it)
    torch.cuda.synchronize()

    # ---- CPU baseline: the reference's beam_search over the same graph, rank 0 at N=1 ------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_search(S["adj_h"], S["start_h"], base.view(n, d).cpu().numpy(), qh.numpy(), chosen, k,
                                  args.cpu_seconds, out_ids, nq, cfg.metric)

    # ---- the build's roofline: its algorithmic bytes (an untimed rebuild whose
    # searches count distinct evaluations, EXACT visited mode) over the timed
    # build's wall time and its kernel time --------------------------------------------------
    build_roof = None
    if build_mode == "single-gpu" and not args.no_build_roofline:
        os.environ["GANN_BUILD_VISITED"] = "exact"
        xi = g.Index.from_device(base.data_ptr(), n, d, cfg.np_dtype, cfg.metric, cfg.R, dev)
        xi.reset_stats()
        xi.build(S["params"])
        torch.cuda.synchronize()
        del os.environ["GANN_BUILD_VISITED"]
        xb = xi.stats()
        same = sha16(xi.export_graph()[0]) == S["graph_sha"]
        xi.close()
        del xi
        bb = build_bytes(xb, n, d * s_el, cfg.R)
        kern_ms = sum(bstats["build_ms"].values())
        build_roof = {
            "bound": "hbm", "unit": "GB/s", "peak": peak,
            "achieved": round(bb["total"] / build_s / 1e9, 1), "frac": round(bb["total"] / build_s / 1e9 / peak, 4),
            "basis": "algorithmic bytes of the whole build (SURVEY.md §8d: per point B_search + |V| d s + 4R, per batch "
                     "16 E + target rows read/written + re-pruned lists' rows) / the timed build's wall time",
            "algorithmic_bytes": {kk: round(v) for kk, v in bb.items()},
            "bytes_per_point": round(bb["total"] / n, 1),
            "kernel_time_frac": round(bb["total"] / (kern_ms / 1e3) / 1e9 / peak, 4) if kern_ms else None,
            "distinct_evals_per_point": round(xb["evaluations"] / n, 1),
            "fast_filter_evals_per_point": round(bstats["evaluations"] / n, 1),
            "exact_count_rebuild_graph_identical": same,
        }

    peak_note = ("algorithmic bytes count each query's rows; rows shared across queries (hubs) are served "
                 "from the 126 MB L2, so achieved can exceed the HBM peak" if achieved > peak else None)
    line = {
        "metric": METRIC,
        "value": round(qps, 1),
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": cfg.dtype,
        "data": "synthetic: seeded Gaussian mixture with BASELINE config shapes (datagen.py), generated in HBM",
        "config": config_obj(args, cfg, nq, chosen, recall),
        "parity": {"graph_sha256": S["graph_sha"], "start": int(S["start_h"]), "ids_sha256": S["ids_sha"],
                   "basis": "sha256[:16] of the n x R uint32 graph rows (GANN_NONE padded) and of the headline "
                            "search's nq x k ids; the reference arm prints the same over graphann's own build "
                            "and search"},
        "streams": nstreams,
        "step_pipelining": ("steps alternate over 2 streams: a step's tail overlaps the next step's start; every "
                            "step searches its whole batch; value = K*nq / elapsed of all K" if nstreams > 1
                            else "serial launches"),
        "roofline": {
            "bound": "hbm",
            "kernel": "search_batch_kernel" if sstats.get("merges", 0) else "search_kernel",  # the batch kernel counts its steps
            "achieved": round(achieved, 1), "peak": peak,
            "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
            "frac_nominal_8tbs": round(achieved / 8000.0, 4),
            "algorithmic_bytes_per_launch": round(per_launch_bytes),
            "avg_launch_ms": round(avg_launch_s * 1e3, 4),
            "launch_ms_basis": ("elapsed of the K pipelined launches / K (sustained)" if nstreams > 1
                                else "mean of the launches' own event spans"),
            "launch_event_span_ms_mean": round(statistics.mean(step_ms), 4),
            "outputs_agree_across_streams": outs_agree,
            "note": peak_note,
            "traffic": traffic_from_profile(cfg.name, chosen),
            "gathered": gathered_obj(sstats, args.steps, d * s_el, nq, k, cfg.R, avg_launch_s, peak,
                                    traffic_from_profile(cfg.name, chosen)),
            "distinct_evals_per_query": round(xstats["evaluations"] / nq, 1),
            "evals_per_query_fast_filter": round(sstats["evaluations"] / (nq * args.steps), 1),
            "expansions_per_query": round(xstats["expansions"] / nq, 1),
            "at_sweep_end": sweep_end,
        },
        "cpu_baseline": cpu,
        "e2e": {"value": round(world * nq * args.steps / e2e_s, 1), "unit": "queries/s",
                "h2d_bytes_per_step": nq * d * s_el, "d2h_bytes_per_step": nq * k * 8,
                "api": f"gann_search_async on {nstreams} stream(s) (pinned host buffers, H2D + search + D2H per step)",
                "ids_match_device_path": e2e_match,
                "blocking": {"value": round(world * nq * args.steps / e2e_block_s, 1),
                             "api": "gann_search (blocking call, pinned host buffers)"}},
        "gpu_launches": args.steps,
        "clocks": clocks,
        "build": {
            "points_per_s": round(n / build_s, 1), "seconds": round(build_s, 3), "mode": build_mode,
            "warmup": "none: one build, including its scratch allocation",
            "phases_ms": {kk: round(v, 1) for kk, v in bstats["build_ms"].items()},
            "mean_degree": round(deg_mean, 3), "replicas_identical": replicas_identical, **S["build_extra"],
            "roofline": build_roof,
            "stats": {kk: v for kk, v in bstats.items() if kk != "build_ms"},
        },
        "qps_curve": {"basis": "recall over all queries; QPS of 4 launches (sweep) / 2 launches (past the sweep) "
                               "timed as the headline",
                      "sweep": curve, "past_sweep": S["ext_curve"],
                      "target_reached": S["target_reached"],
                      "on_chip_beam_limit": S["max_beam"]},
        "secondary_sweep": {"semantics": "reference eval {L, k_gate=10, eps}, top-10, 3 launches timed as the headline",
                            "points": secondary},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _tensor_from_ptr(ptr, nbytes):
    """A torch uint8 view of device memory owned by the index."""
    import torch

    class _Holder:
        def __init__(self, p, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (p, False), "version": 3}

    return torch.as_tensor(_Holder(ptr, nbytes), device="cuda")


def groundtruth_wide_f32(torch, X, Q, metric, depth, pre=64, chunk=200_000):
    """compute_groundtruth (src/dataset.cpp:172-217) for wide f32 rows, setup
    only: an fp32 GEMM (TF32 off) keeps the best `pre` candidates per query,
    then those are re-scored in the reference's order (sequential over the
    dimensions, each multiply and add rounded separately: src/metric.cpp:38-59)
    and sorted by (dist, id). A true top-`depth` id would have to lose more
    than `pre - depth` places to GEMM rounding to be missed."""
    torch.backends.cuda.matmul.allow_tf32 = False
    nq, n = Q.shape[0], X.shape[0]
    best_s = torch.full((nq, pre), float("inf"), device="cuda")
    best_i = torch.zeros((nq, pre), dtype=torch.int64, device="cuda")
    qn = (Q * Q).sum(1, keepdim=True)
    for p0 in range(0, n, chunk):
        xc = X[p0:p0 + chunk]
        sc = -(Q @ xc.T) if metric == "ip" else qn + (xc * xc).sum(1)[None, :] - 2.0 * (Q @ xc.T)
        vals, ids = torch.topk(sc, min(pre, sc.shape[1]), dim=1, largest=False)
        cat_s = torch.cat([best_s, vals], 1)
        cat_i = torch.cat([best_i, ids + p0], 1)
        sel = torch.topk(cat_s, pre, dim=1, largest=False).indices
        best_s, best_i = torch.gather(cat_s, 1, sel), torch.gather(cat_i, 1, sel)
    cand = X[best_i]  # (nq, pre, d)
    acc = torch.zeros((nq, pre), device="cuda")
    for j in range(Q.shape[1]):  # elementwise ops round separately: mul, then add
        if metric == "ip":
            acc = acc + Q[:, j:j + 1] * cand[:, :, j]
        else:
            diff = Q[:, j:j + 1] - cand[:, :, j]
            acc = acc + diff * diff
    dist_ = -acc if metric == "ip" else acc
    dh, ih = dist_.cpu().numpy(), best_i.cpu().numpy()
    order = np.lexsort((ih, dh), axis=1)[:, :depth]
    return (np.take_along_axis(ih, order, 1).astype(np.uint32), np.take_along_axis(dh, order, 1).astype(np.float32))


def cpu_baseline_search(adj, start, data, q_host, L, k, seconds, out_ids, nq, metric="l2"):
    """graphann's beam_search (oracle/_ref, all host threads) over our graph,
    the same queries and beam: a bounded ~10 s sample beside the GPU number."""
    from oracle.oracle import Oracle, available
    kind = "reference" if available("ref") else "port"
    orc = Oracle("ref" if kind == "reference" else "orc")
    secs, ids, reps = orc.time_search(adj, start, data, q_host, L, L, 0.0, k_out=k, metric=metric, workers=0,
                                      reps=1, min_seconds=seconds)
    gpu_ids = out_ids.cpu().numpy().view(np.uint32).reshape(nq, k)
    cores = os.cpu_count()
    return {"value": round(nq / secs, 1), "unit": "queries/s", "cores": cores, "kind": kind,
            "sample": f"all {nq} queries per pass, best of {reps} passes (>= {seconds:.0f} s), beam {{L={L},L,0}} over "
                      f"the same {len(adj)}-point graph, parallel_for over queries on {cores} threads",
            "ids_identical_to_gpu": float((ids == gpu_ids).all(axis=1).mean())}


def host_points(cfg, n):
    """The config's first n points on the host (numpy; bit-identical to the
    device generator the GPU arm uses). u8 configs on a thread pool."""
    if cfg.dtype == "f32":
        out = np.empty((n, cfg.d), np.float32)
        for r0 in range(0, n, 200_000):  # bounded float64 temporaries
            r1 = min(n, r0 + 200_000)
            out[r0:r1] = datagen.gen_f32_numpy(r1 - r0, cfg.d, cfg.clusters, cfg.sigma, cfg.norm_sigma, 0.0,
                                               cfg.center_seed, cfg.base_seed, row0=r0)
        return out
    return datagen.host_base_parallel(cfg, n)


# ---------------------------------------------------------------------------------
def run_reference(args):
    """The reference's own CPU path, end to end, on this arm's workload: the
    config's points regenerated on the host (no GPU, no import of our
    package), graphann's build loop over them (build_diskann's prefix-doubling
    batches with the config's cap: src/diskann.cpp:31-70), graphann's
    compute_groundtruth (src/dataset.cpp:172-217), and graphann's beam_search
    timed per step over all queries with parallel_for on every host thread
    (measure_qps, src/eval.cpp:57-101). The beam is chosen by the same rule as
    our arm from graphann's own recall curve. Under torchrun only rank 0 runs."""
    if int(os.environ.get("RANK", 0)) != 0:
        return
    from oracle.oracle import Oracle, available

    kind = "reference" if available("ref") else "port"
    orc = Oracle("ref" if kind == "reference" else "orc")
    cfg, nq = workload(args)
    k = cfg.k
    cores = os.cpu_count()
    prefix = args.ref_build == "prefix"
    n = min(args.ref_n, cfg.n) if prefix else cfg.n
    t0 = time.perf_counter()
    data = host_points(cfg, n)
    queries = datagen.host_queries(cfg, nq)
    gen_s = time.perf_counter() - t0
    # ---- graphann's build (timed) ---------------------------------------------------------
    cap = (int(n * cfg.batch_cap_frac) if cfg.batch_cap_frac else 0) if prefix else cfg.max_batch
    t0 = time.perf_counter()
    adj, start = orc.build(data, cfg.R, cfg.L, cfg.alpha, metric=cfg.metric, cap=cap, workers=0)
    build_s = time.perf_counter() - t0
    graph_sha = sha16(adj)
    # ---- graphann's ground truth ------------------------------------------------------------
    t0 = time.perf_counter()
    gt_ids, gt_d = orc.groundtruth(data, queries, GT_DEPTH, metric=cfg.metric, workers=0)
    gt_s = time.perf_counter() - t0

    def one_pass(L, q=queries):
        sec, ids, _ = orc.time_search(adj, start, data, q, L, L, 0.0, k_out=k, metric=cfg.metric, workers=0, reps=1)
        return sec, ids

    def recall_of(ids, rows=None):
        ti, td = (gt_ids, gt_d) if rows is None else (gt_ids[:rows], gt_d[:rows])
        return float(evalutil.recall_at_k(ti, td, ids if rows is None else ids[:rows], k).mean())

    # ---- QPS / recall at every beam of the sweep (one pass each), the headline beam -----------
    curve = []
    for L in sweep_beams(args):
        sec, ids = one_pass(L)
        curve.append({"L": L, "recall@10": round(recall_of(ids), 5), "qps": round(nq / sec, 1),
                      "ms_per_pass": round(1e3 * sec, 2)})

    def eval_L(L):
        sec, ids_l = one_pass(L)
        return recall_of(ids_l), {"qps": round(nq / sec, 1), "ms_per_pass": round(1e3 * sec, 2)}

    chosen, reached, ext = choose_beam(args, curve, eval_L)
    recall = next(c["recall@10"] for c in curve + ext if c["L"] == chosen)
    # ---- timed steps at the headline beam --------------------------------------------------------
    for _ in range(args.warmup):
        one_pass(chosen)
    secs, ids = [], None
    for _ in range(args.steps):
        sec, ids = one_pass(chosen)
        secs.append(sec)
    value = nq * args.steps / sum(secs)
    sample = (f"graphann beam_search {{L={chosen},L,0}} top-{k}, one pass over all {nq} queries per step, over "
              f"graphann's own {n}-point graph of the config (built here), parallel_for on {cores} threads")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 1), "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * sum(secs) / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype,
        "data": "synthetic: seeded Gaussian mixture with BASELINE config shapes (datagen.py numpy restatement, "
                "bit-identical to the device generator)",
        "config": config_obj(args, cfg.scaled(n) if prefix else cfg, nq, chosen, recall),
        "parity": {"graph_sha256": graph_sha, "start": int(start), "ids_sha256": sha16(ids),
                   "basis": "sha256[:16] of graphann's n x R uint32 graph rows (0xFFFFFFFF padded) and of its "
                            "headline search's nq x k ids"},
        "cpu_baseline": {"value": round(value, 1), "unit": "queries/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": round(value, 1), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "build": {"points_per_s": round(n / build_s, 1), "seconds": round(build_s, 3), "n": n, "cores": cores,
                  "batch_cap": cap, "graph_sha256": graph_sha,
                  "sample": ("graphann's build loop over the config's whole point set" if not prefix else
                             f"graphann's build loop over the first {n} points")},
        "setup_seconds": {"generate": round(gen_s, 1), "groundtruth": round(gt_s, 1)},
        "qps_curve": {"basis": "recall and QPS of one pass over all queries per beam",
                      "sweep": curve, "past_sweep": ext, "target_reached": reached},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
