"""Multi-GPU plumbing for the query path (one process per GPU).

Queries shard naturally with the index replicated: rank r
searches its own contiguous block of query rows and there is no data-path
collective. torch.distributed is used only for the barrier, the max-over-ranks
timing and the replica check. Backend-agnostic (nccl on GPUs, gloo in tests).
"""
from __future__ import annotations


def query_rows(rank: int, per_rank: int) -> tuple[int, int]:
    """Rows [row0, row0 + per_rank) of the query stream belong to `rank`."""
    return rank * per_rank, per_rank


def reduce_scalar(x: float, op: str = "max", dist=None, device="cpu") -> float:
    """max / min / sum / mean of a per-rank scalar over all ranks (identity at world 1)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN}.get(op, dist.ReduceOp.SUM))
    v = float(t.item())
    return v / dist.get_world_size() if op == "mean" else v


def replicas_identical(checksum: int, dist=None) -> bool:
    """True when every rank holds the same index (checksums all-gathered)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return True
    sums = [None] * dist.get_world_size()
    dist.all_gather_object(sums, int(checksum))
    return len(set(sums)) == 1
