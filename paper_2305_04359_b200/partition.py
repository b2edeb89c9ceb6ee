"""Vertex-partitioned batch build across GPUs (BASELINE config 4).

One process per GPU. Every rank holds all points; rank r owns graph rows
[r*P, (r+1)*P). ``PartitionedIndex.build_native`` runs the whole batch loop in
C++ (``gann_part_build``) over a ``gann_exchange`` — the library's NCCL
transport (``NcclExchange``) or a torch.distributed one (``DistExchange``);
``build`` drives the same steps from Python. Each build batch:

1. phase 1 (``gann_part_phase1``): the rank inserts the batch points it owns —
   beam search over the whole graph (peers' rows read through CUDA IPC / NVLink
   peer mappings) and robustPrune into its own rows — and groups the reverse
   pairs (target, batch ordinal) by the target's owner;
2. exchange: one all-to-all-v of the pairs (8 bytes each) with
   ``torch.distributed`` (NCCL on GPUs; gloo + host staging in the CPU-side
   test of the same logic);
3. phase 2 (``gann_part_phase2``): the owner merges the received pairs into
   its rows; the merge sorts a group by batch ordinal, which restores the
   single-GPU pair order exactly;
4. barrier: the next batch's searches read every rank's updated rows.

The union of the partitions equals the single-GPU build row for row.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib
from .api import ELEM, METRIC, RULE, DiskannParams, _p


# include/gann.h gann_exchange: the collectives the C++ build loop calls
_COUNTS = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64))
_PAIRS = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p, C.POINTER(C.c_uint64),
                     C.c_void_p)
_BARRIER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)


class GannExchange(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("rank", C.c_uint32), ("nranks", C.c_uint32),
                ("alltoall_counts", _COUNTS), ("alltoallv", _PAIRS), ("barrier", _BARRIER)]


class DistExchange:
    """gann_exchange over a torch.distributed process group: any backend (the
    CPU-side tests use gloo, staging the device pairs through host memory).
    Keeps the ctypes callbacks alive while the build runs."""

    def __init__(self, dist, device: int = 0):
        import torch
        self.dist, self.torch, self.device = dist, torch, device
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.error = None
        self._cb = (_COUNTS(self._counts), _PAIRS(self._pairs), _BARRIER(self._barrier))
        self.struct = GannExchange(None, self.rank, self.world, *self._cb)

    def _guard(self, f):
        try:
            f()
            return 0
        except Exception as e:  # noqa: BLE001 — reported as a failed collective
            self.error = repr(e)
            return 1

    def _counts(self, ctx, send, recv):
        def run():
            t = self.torch
            sc = t.tensor([send[i] for i in range(self.world)], dtype=t.int64)
            rc = t.empty(self.world, dtype=t.int64)
            self.dist.all_to_all_single(rc, sc)
            for i in range(self.world):
                recv[i] = int(rc[i])
        return self._guard(run)

    def _pairs(self, ctx, d_send, sc, d_recv, rc, stream):
        def run():
            t = self.torch
            s = [int(sc[i]) for i in range(self.world)]
            r = [int(rc[i]) for i in range(self.world)]
            send = (_device_view(d_send, sum(s) * 8).view(t.int64).cpu() if sum(s) else t.empty(0, dtype=t.int64))
            recv = t.empty(sum(r), dtype=t.int64)
            self.dist.all_to_all_single(recv, send, r, s)
            if sum(r):
                _device_view(d_recv, sum(r) * 8).view(t.int64).copy_(recv.to(f"cuda:{self.device}"))
            t.cuda.synchronize(self.device)
        return self._guard(run)

    def _barrier(self, ctx, stream):
        return self._guard(lambda: self.dist.barrier())


class NcclExchange:
    """gann_exchange_nccl: the library's NCCL transport (ncclSend/ncclRecv on
    the index's stream). The unique id is made by rank 0 and shared through
    the caller's process group."""

    def __init__(self, dist, device: int = 0):
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            check(lib().gann_nccl_unique_id(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0)
        uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        comm = C.c_void_p()
        check(lib().gann_nccl_comm_init(uid, self.rank, self.world, device, C.byref(comm)))
        self.comm = comm
        self.struct = GannExchange()
        check(lib().gann_exchange_nccl(comm, self.rank, self.world, C.byref(self.struct)))
        self.error = None

    def close(self):
        if getattr(self, "comm", None):
            lib().gann_nccl_comm_destroy(self.comm)
            self.comm = None


class PartitionedIndex:
    """This rank's partition of a vertex-partitioned index."""

    def __init__(self, points, metric: str, degree_bound: int, dist, device: int = 0, shape=None, dtype=None):
        """points: a host array (n, d), or a device pointer with shape=(n, d) and dtype."""
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device
        self.R = degree_bound
        self.metric = metric
        h = C.c_void_p()
        if shape is None:
            points = np.ascontiguousarray(points)
            self.n, self.d = points.shape
            check(lib().gann_index_create_part(_p(points), self.n, self.d, ELEM[points.dtype], METRIC[metric],
                                               degree_bound, self.rank, self.world, device, C.byref(h)))
        else:
            self.n, self.d = shape
            check(lib().gann_index_create_part_device(C.c_void_p(points or None), self.n, self.d, ELEM[np.dtype(dtype)],
                                                      METRIC[metric], degree_bound, self.rank, self.world, device,
                                                      C.byref(h)))
        self._h = h
        base, rows = C.c_uint64(), C.c_uint64()
        check(lib().gann_part_info(h, None, None, C.byref(base), C.byref(rows)))
        self.base, self.rows = base.value, rows.value
        self._attach_peers()

    def _attach_peers(self):
        """Open every peer's rows. A failure on any rank is seen by all ranks
        (``peers_ok``) instead of leaving the others waiting in a collective."""
        handle = (C.c_uint8 * 64)()
        check(lib().gann_part_ipc_handle(self._h, handle))
        handles = [None] * self.world
        self.dist.all_gather_object(handles, bytes(handle))
        ok, self.attach_error = 1, None
        try:
            for r, hb in enumerate(handles):
                if r != self.rank:
                    buf = (C.c_uint8 * 64).from_buffer_copy(hb)
                    check(lib().gann_part_attach(self._h, r, buf))
        except Exception as e:  # noqa: BLE001 — reported through peers_ok
            ok, self.attach_error = 0, str(e)
        oks = [None] * self.world
        self.dist.all_gather_object(oks, ok)
        self.peers_ok = all(oks)

    def close(self):
        if getattr(self, "_h", None):
            lib().gann_index_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def build(self, params: DiskannParams, nccl: bool = False) -> dict:
        import torch
        if not self.peers_ok:
            raise RuntimeError(f"peer rows not mapped on every rank ({self.attach_error})")
        nb = C.c_uint32()
        check(lib().gann_part_build_begin(self._h, params.build_beam, params.alpha, RULE[params.rule], params.seed,
                                          params.max_batch, C.byref(nb)))
        counts = np.zeros(self.world, np.uint64)
        ptr = C.c_void_p()
        exchanged = 0
        dev = torch.device("cuda", self.device)
        for b in range(nb.value):
            check(lib().gann_part_phase1(self._h, b, _p(counts), C.byref(ptr)))
            send_counts = [int(c) for c in counts]
            total = sum(send_counts)
            # pair counts first, then the pairs themselves (int64 = one interleaved pair)
            sc = torch.tensor(send_counts, dtype=torch.int64)
            rc = torch.empty(self.world, dtype=torch.int64)
            if nccl:
                sc, rc = sc.to(dev), rc.to(dev)
            self.dist.all_to_all_single(rc, sc)
            recv_counts = [int(x) for x in rc.cpu().tolist()]
            m = sum(recv_counts)
            send = _device_view(ptr.value, total * 8).view(torch.int64) if total else torch.empty(0, dtype=torch.int64, device=dev)
            if nccl:
                recv = torch.empty(m, dtype=torch.int64, device=dev)
                self.dist.all_to_all_single(recv, send, recv_counts, send_counts)
            else:  # gloo: stage through host memory
                recv_h = torch.empty(m, dtype=torch.int64)
                self.dist.all_to_all_single(recv_h, send.cpu(), recv_counts, send_counts)
                recv = recv_h.to(dev)
            torch.cuda.synchronize(dev)
            check(lib().gann_part_phase2(self._h, b, C.c_void_p(recv.data_ptr() if m else None), m))
            exchanged += total
            self.dist.barrier()  # every rank's rows are final before the next batch searches
        return {"batches": nb.value, "pairs_sent": exchanged}

    def build_native(self, params: DiskannParams, exchange) -> dict:
        """The whole partitioned build in C++ (gann_part_build) with the given
        exchange (DistExchange or NcclExchange)."""
        if not self.peers_ok:
            raise RuntimeError(f"peer rows not mapped on every rank ({self.attach_error})")
        sent = C.c_uint64()
        rc = lib().gann_part_build(self._h, C.byref(exchange.struct), params.build_beam, params.alpha,
                                   RULE[params.rule], params.seed, params.max_batch, C.byref(sent))
        if rc and exchange.error:
            raise RuntimeError(f"exchange failed: {exchange.error}")
        check(rc)
        return {"pairs_sent": sent.value}

    def device_points(self):
        """(pointer, stride) of this index's device points (filled in place when
        the index was created from a NULL pointer)."""
        pts, stride, adj = C.c_void_p(), C.c_uint64(), C.c_void_p()
        check(lib().gann_index_device_ptrs(self._h, C.byref(pts), C.byref(stride), C.byref(adj)))
        return pts.value, stride.value

    def as_index(self):
        """An Index view of this partition's handle (not owning it): its search
        calls read every partition in place."""
        from .api import Index

        class _View(Index):
            def close(self):
                self._h = None

        v = _View.__new__(_View)
        v._init(self._h, self.metric, self.device)
        v._owner = self  # keep the partition alive while the view is used
        return v

    def batch_cap(self, build_beam: int, budget_bytes: int) -> int:
        """gann_part_batch_cap: the largest global batch whose scratch fits."""
        v = C.c_uint32()
        check(lib().gann_part_batch_cap(self._h, build_beam, budget_bytes, C.byref(v)))
        return v.value

    def search_device(self, q_ptr: int, nq: int, params, k_out: int, ids_ptr: int, dists_ptr: int,
                      stream: int = 0) -> None:
        """Beam search over the partitioned graph: every row is read where it
        lives (this GPU's partition, or a peer's through its CUDA IPC / NVLink
        mapping); no replica of the graph is needed."""
        check(lib().gann_search_device(self._h, C.c_void_p(q_ptr), nq, k_out, params.beam, params.k,
                                       params.epsilon, 0, C.c_void_p(ids_ptr), C.c_void_p(dists_ptr), None, None,
                                       C.c_void_p(stream or None)))

    def stats(self) -> dict:
        """This rank's share of the build counters and phase times."""
        from .api import Index
        return Index.stats(self)

    def start(self) -> int:
        s = C.c_uint32()
        check(lib().gann_index_info(self._h, None, None, None, None, None, C.byref(s)))
        return s.value

    def device_rows(self):
        """A torch view (rows * R int32) of this partition's rows on the device."""
        pts, stride, adj = C.c_void_p(), C.c_uint64(), C.c_void_p()
        check(lib().gann_index_device_ptrs(self._h, C.byref(pts), C.byref(stride), C.byref(adj)))
        import torch
        return _device_view(adj.value, self.rows * self.R * 4).view(torch.int32)

    def export_rows(self):
        """This partition's rows (rows x R) and the start vertex."""
        adj = np.empty((self.rows, self.R), np.uint32)
        deg = np.empty(self.rows, np.uint32)
        s = C.c_uint32()
        check(lib().gann_export_graph(self._h, _p(adj), _p(deg), C.byref(s)))
        return adj, s.value


def _device_view(ptr: int, nbytes: int):
    import torch

    class _Holder:
        def __init__(self, p, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (p, False), "version": 3}

    return torch.as_tensor(_Holder(ptr, nbytes), device="cuda")
