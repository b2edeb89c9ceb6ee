"""ctypes binding of ``libgann_b200.so`` — the C ABI declared in ``include/gann.h``.

The library is built in-tree (``paper_2305_04359_b200/libgann_b200.so``) by
``__graft_entry__.build()``. There is no fallback: if the shared object is
missing, importing the package fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libgann_b200.so"
if os.environ.get("GANN_LIB"):  # experiments: an alternative in-tree build of the same ABI
    LIB_PATH = HERE / os.environ["GANN_LIB"]

GANN_NONE = 0xFFFFFFFF
GANN_OK, GANN_EINVAL, GANN_EIO, GANN_ECUDA = 0, 1, 2, 3


class GannError(RuntimeError):
    """A CUDA-side failure (GANN_ECUDA)."""


class GannStats(C.Structure):
    _fields_ = [
        ("queries", C.c_uint64),
        ("expansions", C.c_uint64),
        ("evaluations", C.c_uint64),
        ("filter_drops", C.c_uint64),
        ("adj_entries", C.c_uint64),
        ("prune_lists", C.c_uint64),
        ("prune_candidates", C.c_uint64),
        ("prune_evals", C.c_uint64),
        ("back_pairs", C.c_uint64),
        ("back_groups", C.c_uint64),
        ("back_pruned", C.c_uint64),
        ("build_ms", C.c_double * 6),
        ("merges", C.c_uint64),
        ("survivors", C.c_uint64),
        ("moved", C.c_uint64),
        ("duplicates", C.c_uint64),
        ("guess_hits", C.c_uint64),
    ]


# name -> (restype, argtypes); the signatures of include/gann.h
_u32, _u64, _i, _f, _vp = C.c_uint32, C.c_uint64, C.c_int, C.c_float, C.c_void_p
_pp = C.POINTER(C.c_void_p)
SIGNATURES = {
    "gann_last_error": (C.c_char_p, []),
    "gann_version": (C.c_char_p, []),
    "gann_index_create": (_i, [_vp, _u64, _u32, _i, _i, _u32, _i, _pp]),
    "gann_index_create_device": (_i, [_vp, _u64, _u32, _i, _i, _u32, _i, _pp]),
    "gann_index_free": (None, [_vp]),
    "gann_index_info": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "gann_build": (_i, [_vp, _u32, _f, _i, _u64, _u32]),
    "gann_build_diskann": (_i, [_vp, _u64, _u32, _i, _i, _u32, _u32, _f, _i, _u64, _u32, _i, _pp]),
    "gann_import_graph": (_i, [_vp, _vp, _u32]),
    "gann_export_graph": (_i, [_vp, _vp, _vp, _vp]),
    "gann_search": (_i, [_vp, _vp, _u32, _u32, _u32, _u32, _f, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _u32]),
    "gann_search_device": (_i, [_vp, _vp, _u32, _u32, _u32, _u32, _f, _i, _vp, _vp, _vp, _vp, _vp]),
    "gann_stage_queries": (_i, [_vp, _vp, _u32]),
    "gann_search_max_beam": (_i, [_vp, C.POINTER(C.c_uint32)]),
    "gann_debug_check": (_i, [_i, _vp, _vp]),
    "gann_search_staged": (_i, [_vp, _u32, _u32, _u32, _f, _vp, _vp, _vp]),
    "gann_search_async_scratch": (_u64, [_vp, _u32, _u32]),
    "gann_search_async": (_i, [_vp, _vp, _u32, _u32, _u32, _u32, _f, _vp, _vp, _vp, _u64, _vp]),
    "gann_alpha_prune": (_i, [_vp, _vp, _vp, _u32, _vp, _vp, _f, _i, _vp, _vp]),
    "gann_group_by_key": (_i, [_vp, _vp, _u64, _i, _vp, _vp, _vp, _vp]),
    "gann_choose_start": (_i, [_vp, _vp]),
    "gann_insert_batch": (_i, [_vp, _vp, _u32, _u32, _f, _i, _vp]),
    "gann_apply_back_edges": (_i, [_vp, _vp, _vp, _u64, _f, _i]),
    "gann_shuffled_order": (None, [_u32, _u64, _u32, _vp]),
    "gann_shuffle_swap_log": (None, [_u32, _u64, _vp]),
    "gann_batch_ranges": (_u32, [_u64, _u32, _vp, _vp, _u32]),
    "gann_insert_seed": (_u64, [_u64]),
    "gann_groundtruth": (_i, [_vp, _vp, _u32, _u32, _vp, _vp]),
    "gann_groundtruth_device": (_i, [_vp, _vp, _u32, _u32, _vp, _vp, _vp]),
    "gann_generate_u8": (_i, [_vp, _u64, _u32, _u32, _f, _f, _u64, _u64, _u64, _i]),
    "gann_generate_f32": (_i, [_vp, _u64, _u32, _u32, _f, _f, _f, _u64, _u64, _u64, _i]),
    "gann_normal_table": (_i, [_vp]),
    "gann_save_graph": (_i, [_vp, C.c_char_p]),
    "gann_load_graph": (_i, [_vp, C.c_char_p]),
    "gann_index_create_from_file": (_i, [C.c_char_p, _i, _u32, _i, _pp]),
    "gann_range_search": (_i, [_vp, _vp, _u32, _f, _u32, _f, _u32, _vp, _vp, _vp]),
    "gann_hnsw_create": (_i, [_vp, _u32, _vp, _u32, _u32, _pp]),
    "gann_hnsw_search": (_i, [_vp, _vp, _u32, _u32, _u32, _u32, _f, _i, _vp, _vp, _vp, _vp]),
    "gann_hnsw_free": (None, [_vp]),
    "gann_index_create_part": (_i, [_vp, _u64, _u32, _i, _i, _u32, _u32, _u32, _i, _pp]),
    "gann_index_create_part_device": (_i, [_vp, _u64, _u32, _i, _i, _u32, _u32, _u32, _i, _pp]),
    "gann_import_graph_device": (_i, [_vp, _vp, _u32]),
    "gann_part_info": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "gann_part_ipc_handle": (_i, [_vp, _vp]),
    "gann_part_attach": (_i, [_vp, _u32, _vp]),
    "gann_part_build_begin": (_i, [_vp, _u32, _f, _i, _u64, _u32, _vp]),
    "gann_part_phase1": (_i, [_vp, _u32, _vp, _pp]),
    "gann_part_phase2": (_i, [_vp, _u32, _vp, _u64]),
    "gann_part_build": (_i, [_vp, _vp, _u32, _f, _i, _u64, _u32, _vp]),
    "gann_part_batch_cap": (_i, [_vp, _u32, _u64, _vp]),
    "gann_nccl_unique_id": (_i, [_vp]),
    "gann_nccl_comm_init": (_i, [_vp, _u32, _u32, _i, _pp]),
    "gann_nccl_comm_destroy": (_i, [_vp]),
    "gann_exchange_nccl": (_i, [_vp, _u32, _u32, _vp]),
    "gann_get_stats": (_i, [_vp, C.POINTER(GannStats)]),
    "gann_reset_stats": (_i, [_vp]),
    "gann_release_scratch": (_i, [_vp]),
    "gann_index_device_ptrs": (_i, [_vp, _pp, C.POINTER(C.c_uint64), _pp]),
}

_lib = None


def lib() -> C.CDLL:
    """Load the in-tree shared object (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == GANN_OK:
        return
    msg = lib().gann_last_error().decode()
    if rc == GANN_EINVAL:
        raise ValueError(msg)
    if rc == GANN_EIO:
        raise IOError(msg)
    raise GannError(msg)
