"""ctypes binding of libpbsa_b200.so (include/pbsa_b200.h).

This is exactly the binding a reference-side maintainer would add; the
Python API in `pbsa.py` is layered on top of it.  There is no fallback: if the shared library is
missing or fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PBSA_LIB_PATH: perf experiments only (e.g. the -DPBSA_K3_TRACE build of `make trace-lib`)
LIB_PATH = os.environ.get("PBSA_LIB_PATH") or os.path.join(HERE, "_lib", "libpbsa_b200.so")

PBSA_OK, PBSA_EINVAL, PBSA_ECUDA, PBSA_EUNSUPPORTED = 0, 1, 2, 3
MODE_DENOISE, MODE_CACHE_UPDATE = 0, 1

_vp, _i32, _i64, _f32 = C.c_void_p, C.c_int, C.c_int64, C.c_float


class MemInfo(C.Structure):
    _fields_ = [
        ("units", _i32), ("capacity_c", _i32), ("window_chunks", _i32),
        ("blocks_per_chunk", _i32), ("b", _i32), ("d", _i32), ("n_slots", _i32),
        ("n_p", _i32), ("n_sinks", _i32), ("n_l", _i32), ("chunks_committed", _i64),
        ("k_pool", _vp), ("v_pool", _vp), ("krep", _vp), ("dense_slots", _vp),
        ("local_slots", _vp), ("key_slots", _vp), ("stage_slots", _vp), ("p_ids", _vp),
        ("p_scores", _vp), ("l_ids", _vp), ("dense_stride", _i32), ("local_stride", _i32),
        ("key_stride", _i32),
    ]


class LatentGeom(C.Structure):
    """pbsa_latent_geom: chunk latents [batch][T][H][W][heads*head_dim] blocked by (B_t, B_h, B_w)."""
    _fields_ = [("batch", _i32), ("t", _i32), ("h", _i32), ("w", _i32), ("heads", _i32),
                ("head_dim", _i32), ("block_t", _i32), ("block_h", _i32), ("block_w", _i32)]


class BsaPlan(C.Structure):
    """pbsa_bsa_plan: how the last K3 launch of this thread was planned."""
    _fields_ = [("list_entry_bytes", _i32), ("ctas_per_sm", _i32), ("grid", _i32), ("schedule", _i32),
                ("gangs", _i32), ("max_list", _i32), ("n_tiles", _i32), ("smem_bytes", C.c_size_t)]


SCHED_WHOLE_TILES, SCHED_STREAM_K, SCHED_UNIT_GANGS = 0, 1, 2

_SIGS = {
    "pbsa_last_error": (C.c_char_p, []),
    "pbsa_version": (_i32, []),
    "pbsa_compress": (_i32, [_vp, _i64, _i64, _vp, _i32, _i32, _i32, _i32, _vp, _i64, _vp]),
    "pbsa_score_select_workspace": (C.c_size_t, [_i32, _i32, _i32]),
    "pbsa_score_select": (_i32, [_vp, _vp, _i64, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                                 _i32, _f32, _vp, _vp, _vp, C.c_size_t, _vp]),
    "pbsa_bsa_fwd_workspace": (C.c_size_t, [_i32, _i32, _i32]),
    "pbsa_bsa_fwd": (_i32, [_vp, _vp, _vp, _i32, _vp, _i32, _i32, _vp, _i32, _i32, _vp, _i32,
                            _i32, _i32, _i32, _i32, _f32, _vp, _vp, _vp, C.c_size_t, _vp]),
    "pbsa_bsa_fwd_last_plan": (_i32, [C.POINTER(BsaPlan)]),
    "pbsa_matmul": (_i32, [_vp, _vp, _i32, _i32, _i32, _i32, _f32, _vp, _vp]),
    "pbsa_masked_softmax_rows": (_i32, [_vp, _vp, _i32, _i32, _vp, _vp, _vp]),
    "pbsa_aggregate_scores": (_i32, [_vp, _i32, _i32, _vp, _vp]),
    "pbsa_compress_f32": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp]),
    "pbsa_select_topk_workspace": (C.c_size_t, [_i32, _i32]),
    "pbsa_select_topk": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp, C.c_size_t, _vp, _vp]),
    "pbsa_blockify": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _i32, _vp]),
    "pbsa_topc_select": (_i32, [_vp, _vp, _i32, _i32, _vp, _vp, _vp]),
    "pbsa_dev_alloc": (_i32, [C.POINTER(_vp), C.c_size_t]),
    "pbsa_dev_free": (_i32, [_vp]),
    "pbsa_stream_sync": (_i32, [_vp]),
    "pbsa_bsa_bwd_workspace": (C.c_size_t, [_i32, _i32, _i32, _i32]),
    "pbsa_bsa_bwd": (_i32, [_vp, _vp, _vp, _i32, _vp, _i32, _i32, _vp, _i32, _i32, _vp, _i32,
                            _i32, _i32, _i32, _i32, _f32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, C.c_size_t, _vp]),
    "pbsa_mem_create": (_i32, [C.POINTER(_vp), _i32, _i32, _i32, _i32, _i32, _i32]),
    "pbsa_mem_destroy": (_i32, [_vp]),
    "pbsa_mem_reset": (_i32, [_vp, _vp]),
    "pbsa_mem_get_info": (_i32, [_vp, C.POINTER(MemInfo)]),
    "pbsa_mem_write_chunk": (_i32, [_vp, _vp, _vp, _vp]),
    "pbsa_mem_commit": (_i32, [_vp, _vp, _vp]),
    "pbsa_attend": (_i32, [_vp, _vp, _i32, _f32, _i32, _vp, _vp, _vp]),
    "pbsa_attend_qkv": (_i32, [_vp, _vp, _vp, _vp, _i32, _f32, _i32, _vp, _vp, _vp]),
    "pbsa_attend_qkv_host": (_i32, [_vp, _vp, _vp, _vp, _i32, _f32, _i32, _vp, _vp]),
    "pbsa_mem_host_sync": (_i32, [_vp]),
    "pbsa_mem_host_reserve": (_i32, [_vp]),
    "pbsa_attend_part_ingest": (_i32, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "pbsa_attend_part": (_i32, [_vp, _vp, _i32, _i32, _vp, _i32, _f32, _i32, _vp, _vp, _vp]),
    "pbsa_last_selection_rows": (_i32, [_vp, C.POINTER(_i32)]),
    "pbsa_last_tile_pairs": (_i32, [_vp, C.POINTER(_vp), C.POINTER(_i32)]),
    "pbsa_pair_tiles": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "pbsa_launch_count": (C.c_longlong, []),
    "pbsa_latent_blocks": (_i32, [C.POINTER(LatentGeom), C.POINTER(_i32), C.POINTER(_i32)]),
    "pbsa_attend_latent": (_i32, [_vp, _vp, _vp, _vp, C.POINTER(LatentGeom), _i32, _f32, _i32, _vp, _vp, _vp]),
    "pbsa_last_selection": (_i32, [_vp, C.POINTER(_vp), C.POINTER(_i32), C.POINTER(_vp),
                                   C.POINTER(_i32)]),
    "pbsa_mem_profile": (_i32, [_vp, _i32, _i32]),
    "pbsa_mem_profile_read": (_i32, [_vp, C.POINTER(C.c_double), C.POINTER(_i32), C.POINTER(_i32)]),
    "pbsa_mem_status": (_i32, [_vp, C.POINTER(_i32), _vp]),
    "pbsa_copy": (_i32, [_vp, _vp, C.c_size_t, _vp]),
    "pbsa_pbt1_write": (_i32, [C.c_char_p, _vp, _i32, C.POINTER(C.c_uint64)]),
    "pbsa_pbt1_info": (_i32, [C.c_char_p, C.POINTER(_i32), C.POINTER(C.c_uint64), _i32]),
    "pbsa_pbt1_read": (_i32, [C.c_char_p, _vp, C.c_uint64]),
    "pbsa_pbt1_load_bf16": (_i32, [C.c_char_p, _vp, C.c_uint64, _vp]),
}

# test / experiment hooks (include/pbsa_b200_debug.h) -- not part of the drop-in boundary
_DEBUG_SIGS = {
    "pbsa_debug_tile": (_i32, [_vp, _vp, _vp, _i32, _vp, _vp, _vp]),
    "pbsa_debug_set_fault": (_i32, [C.c_char_p]),
    "pbsa_debug_trace_buffer": (None, [_vp]),
    "pbsa_debug_bwd_trace_buffer": (None, [_vp]),
}

EXPORTED = sorted(_SIGS)
DEBUG_EXPORTED = sorted(_DEBUG_SIGS)


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA library first (`make` or "
            f"`python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")
    lib = C.CDLL(path)
    for name, (res, args) in list(_SIGS.items()) + list(_DEBUG_SIGS.items()):
        if path != os.path.join(HERE, "_lib", "libpbsa_b200.so") and not hasattr(lib, name):
            continue  # an older experiment build (PBSA_LIB_PATH) may predate some entry points
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = load()


class PbsaError(ValueError):
    """Invalid argument / unsupported shape (the reference raises std::invalid_argument)."""


class PbsaCudaError(RuntimeError):
    """CUDA / launch failure."""


def check(rc: int) -> None:
    if rc == PBSA_OK:
        return
    msg = LIB.pbsa_last_error().decode()
    if rc == PBSA_ECUDA:
        raise PbsaCudaError(msg)
    raise PbsaError(msg)
