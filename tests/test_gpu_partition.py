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
