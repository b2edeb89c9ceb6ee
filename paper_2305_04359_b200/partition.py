"""Vertex-partitioned batch build across GPUs (BASELINE config 4).

One process per GPU. Every rank holds all points; rank r owns graph rows
[r*P, (r+1)*P). Each build batch:

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


class PartitionedIndex:
    """This rank's partition of a vertex-partitioned index."""

    def __init__(self, points, metric: str, degree_bound: int, dist, device: int = 0, shape=None, dtype=None):
        """points: a host array (n, d), or a device pointer with shape=(n, d) and dtype."""
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device
        self.R = degree_bound
        h = C.c_void_p()
        if shape is None:
            points = np.ascontiguousarray(points)
            self.n, self.d = points.shape
            check(lib().gann_index_create_part(_p(points), self.n, self.d, ELEM[points.dtype], METRIC[metric],
                                               degree_bound, self.rank, self.world, device, C.byref(h)))
        else:
            self.n, self.d = shape
            check(lib().gann_index_create_part_device(C.c_void_p(points), self.n, self.d, ELEM[np.dtype(dtype)],
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
