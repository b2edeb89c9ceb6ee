"""Vertex-partitioned build: 2 and 3 ranks as separate processes
sharing cuda:0 (peer rows through CUDA IPC, pairs exchanged with gloo
all-to-all-v) must produce the single-GPU graph row for row. The kernels of
different ranks never wait on one another: ranks meet only at host-side
collectives between launches."""
import os
import socket

import numpy as np
import pytest

from helpers import mixture

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, data, params, q):
    import torch.distributed as dist

    import paper_2305_04359_b200 as g
    from paper_2305_04359_b200.partition import PartitionedIndex
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pidx = PartitionedIndex(data, "l2", params["R"], dist, device=0)
    info = pidx.build(g.DiskannParams(params["R"], params["L"], params["alpha"], max_batch=params["cap"]))
    rows, start = pidx.export_rows()
    q.put((rank, pidx.base, rows, start, info))
    dist.barrier()
    pidx.close()
    dist.destroy_process_group()


def _rank_main_device(rank, world, port, data, params, q):
    """bench.py's N>1 path: points from device memory, partitioned build, rows
    gathered into every rank's full replica (gann_import_graph_device)."""
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_2305_04359_b200 as g
    from paper_2305_04359_b200._lib import check, lib
    from paper_2305_04359_b200.partition import PartitionedIndex
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    base = torch.from_numpy(data).cuda()
    n, d = data.shape
    pidx = PartitionedIndex(base.data_ptr(), "l2", params["R"], dist, device=0, shape=(n, d), dtype=np.uint8)
    assert pidx.peers_ok
    pidx.build(g.DiskannParams(params["R"], params["L"], params["alpha"], max_batch=params["cap"]))
    P = -(-n // world)
    rows = torch.full((P * params["R"],), -1, dtype=torch.int32, device="cuda")
    rows[: pidx.rows * params["R"]] = pidx.device_rows()
    parts = [torch.empty(P * params["R"], dtype=torch.int32) for _ in range(world)]
    dist.all_gather(parts, rows.cpu())  # gloo: host staging; NCCL gathers on the device
    full = torch.cat(parts).cuda()
    idx = g.Index.from_device(base.data_ptr(), n, d, np.uint8, "l2", params["R"], 0)
    check(lib().gann_import_graph_device(idx._h, ctypes.c_void_p(full.data_ptr()), pidx.start()))
    adj, _, start = idx.export_graph()
    q.put((rank, adj, start))
    dist.barrier()
    idx.close()
    pidx.close()
    dist.destroy_process_group()


def _spawn(target, world, data, params):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, data, params, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(out, key=lambda x: x[0])


def test_partitioned_build_gathered_replicas():
    import paper_2305_04359_b200 as g
    data = mixture(62, 3000, 32, clusters=10)
    params = {"R": 20, "L": 40, "alpha": 1.2, "cap": 120}
    want = g.build_diskann(data, "l2", g.DiskannParams(20, 40, 1.2, max_batch=120))
    wadj, _, wstart = want.export_graph()
    want.close()
    for rank, adj, start in _spawn(_rank_main_device, 2, data, params):
        assert start == wstart and (adj == wadj).all(), rank


@pytest.mark.parametrize("world,cap", [(2, 0), (3, 150)])
def test_partitioned_build_equals_single_gpu(world, cap):
    import torch.multiprocessing as mp

    import paper_2305_04359_b200 as g
    data = mixture(61, 4000, 32, clusters=12)
    params = {"R": 24, "L": 48, "alpha": 1.2, "cap": cap}
    want = g.build_diskann(data, "l2", g.DiskannParams(24, 48, 1.2, max_batch=cap))
    wadj, _, wstart = want.export_graph()
    want.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, data, params, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    parts.sort(key=lambda x: x[0])
    got = np.concatenate([x[2] for x in parts])
    assert all(x[3] == wstart for x in parts)
    assert got.shape == wadj.shape
    assert (got == wadj).all(), f"{int((got != wadj).any(axis=1).sum())} rows differ"
    assert sum(x[4]["pairs_sent"] for x in parts) > 0


def _rank_main_native(rank, world, port, data, params, q):
    """The C++ build loop (gann_part_build) over a torch.distributed/gloo
    exchange, then a search over the partitioned graph (peer rows through
    CUDA IPC, no replica)."""
    import torch
    import torch.distributed as dist

    import paper_2305_04359_b200 as g
    from paper_2305_04359_b200.partition import DistExchange, NcclExchange, PartitionedIndex
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pidx = PartitionedIndex(data, "l2", params["R"], dist, device=0)
    x = NcclExchange(dist, 0) if params.get("nccl") else DistExchange(dist, 0)
    info = pidx.build_native(g.DiskannParams(params["R"], params["L"], params["alpha"], max_batch=params["cap"]), x)
    rows, start = pidx.export_rows()
    qs = torch.from_numpy(params["queries"]).cuda()
    nq, k = qs.shape[0], 10
    ids = torch.empty(nq * k, dtype=torch.int32, device="cuda")
    ds = torch.empty(nq * k, dtype=torch.float32, device="cuda")
    pidx.search_device(qs.data_ptr(), nq, g.SearchParams(32, 32, 0.0), k, ids.data_ptr(), ds.data_ptr())
    torch.cuda.synchronize()
    q.put((rank, pidx.base, rows, start, info, ids.cpu().numpy().view(np.uint32).reshape(nq, k)))
    dist.barrier()
    if params.get("nccl"):
        x.close()
    pidx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,cap,nccl", [(2, 0, False), (3, 140, False), (1, 100, True)])
def test_native_partitioned_build(world, cap, nccl):
    """gann_part_build (C++ batch loop behind the C ABI) == the single-GPU
    build row for row, over gloo (2-3 ranks sharing cuda:0) and over the
    library's NCCL transport (1 rank: a single-GPU pool cannot host two NCCL
    ranks); the partitioned search returns the single-GPU search's ids."""
    import paper_2305_04359_b200 as g
    data, qs = mixture(63, 3500, 32, clusters=12, nq=64)
    params = {"R": 24, "L": 48, "alpha": 1.2, "cap": cap, "nccl": nccl, "queries": qs}
    want = g.build_diskann(data, "l2", g.DiskannParams(24, 48, 1.2, max_batch=cap))
    wadj, _, wstart = want.export_graph()
    wids = want.search(qs, g.SearchParams(32, 32, 0.0), k_out=10).ids
    want.close()
    parts = _spawn(_rank_main_native, world, data, params)
    got = np.concatenate([x[2] for x in parts])
    assert all(x[3] == wstart for x in parts)
    assert (got == wadj).all(), f"{int((got != wadj).any(axis=1).sum())} rows differ"
    assert world == 1 or sum(x[4]["pairs_sent"] for x in parts) > 0
    for x in parts:
        assert (x[5] == wids).all(), f"rank {x[0]}: partitioned search ids differ"


def test_part_batch_cap_shrinks_with_budget():
    """gann_part_batch_cap: the batch cap grows with the scratch budget and
    shrinks with the beam; at 1B points / 8 GPUs with ~12 GB of room it lands
    in SURVEY.md §8e's 0.2-0.5% of n."""
    import ctypes as C

    from paper_2305_04359_b200._lib import check, lib
    h = C.c_void_p()
    data = mixture(64, 1000, 16, clusters=4)
    check(lib().gann_index_create_part(data.ctypes.data, 1000, 16, 0, 0, 64, 0, 8, 0, C.byref(h)))
    try:
        caps = []
        for budget, L in [(4 << 30, 128), (12 << 30, 128), (12 << 30, 256)]:
            v = C.c_uint32()
            check(lib().gann_part_batch_cap(h, L, budget, C.byref(v)))
            caps.append(v.value)
        assert caps[0] == 1000  # capped at n
        with pytest.raises(ValueError):
            check(lib().gann_part_batch_cap(h, 128, 1 << 20, C.byref(C.c_uint32())))
    finally:
        lib().gann_index_free(h)
