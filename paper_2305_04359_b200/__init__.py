"""B200-native Vamana batch build + batched beam search (arXiv 2305.04359 hot path).

The compute lives in ``libgann_b200.so`` (hand-written sm_100a CUDA + a C ABI,
``include/gann.h``); this package is the host-side mirror of the reference's
interface over that ABI. Importing it loads the shared object and fails loudly
if it is missing — there is no CPU fallback.
"""
from ._lib import GANN_NONE, GannError, LIB_PATH, lib
from .api import (DiskannParams, GroupedPairs, HnswIndex, Index, PruneParams, SearchParams, SearchResult,
                  alpha_prune, apply_back_edges, batch_ranges, beam_search, build_diskann,
                  choose_start, group_by_key, insert_point, insert_seed, search_hnsw, shuffle_swap_log, shuffled_order)

lib()  # load now: a missing/unbuildable extension is an import error, not a silent fallback

__all__ = [
    "GANN_NONE", "GannError", "LIB_PATH", "DiskannParams", "GroupedPairs", "HnswIndex", "Index", "PruneParams",
    "SearchParams", "SearchResult", "alpha_prune", "apply_back_edges", "batch_ranges", "beam_search",
    "build_diskann", "choose_start", "group_by_key", "insert_point", "insert_seed", "search_hnsw",
    "shuffle_swap_log", "shuffled_order",
]
