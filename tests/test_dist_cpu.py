"""CPU: the multi-rank query path with world_size 2 over gloo (127.0.0.1)."""
import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2305_04359_b200 import distutil
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {
        "rows": distutil.query_rows(rank, 10_000),
        "max": distutil.reduce_scalar(1.0 + rank, "max", dist),
        "sum": distutil.reduce_scalar(1.0 + rank, "sum", dist),
        "mean": distutil.reduce_scalar(0.9 + 0.1 * rank, "mean", dist),
        "same": distutil.replicas_identical(12345, dist),
        "diff": distutil.replicas_identical(rank, dist),
    }
    q.put((rank, out))
    dist.destroy_process_group()


def test_two_rank_query_sharding_and_reductions():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (a0, n0), (a1, n1) = res[0]["rows"], res[1]["rows"]
    assert a0 + n0 == a1 and n0 == n1 == 10_000  # disjoint, contiguous shards
    for r in (0, 1):
        assert res[r]["max"] == 2.0 and res[r]["sum"] == 3.0
        assert res[r]["mean"] == pytest.approx(0.95)
        assert res[r]["same"] is True and res[r]["diff"] is False


def test_single_rank_is_identity():
    from paper_2305_04359_b200 import distutil
    assert distutil.reduce_scalar(3.5) == 3.5
    assert distutil.replicas_identical(7)
