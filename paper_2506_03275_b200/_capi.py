"""ctypes binding of the C ABI declared in ``include/csd_b200.h``.

Loads the in-tree ``libcsd_b200.so``.  There is no fallback: if the library is
missing or cannot load, importing the product API raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.path.join(PKG, "libcsd_b200.so")
HEADER = os.path.join(ROOT, "include", "csd_b200.h")

# csd_status / csd_mode / csd_layout
OK, ERR_SHAPE, ERR_INDEX, ERR_NUMERIC, ERR_STATE, ERR_VALUE, ERR_CONFIG, ERR_CUDA, ERR_UNSUPPORTED = range(9)
MODE_CHECK, MODE_PROD = 0, 1
LAYOUT_BHNE, LAYOUT_BNHE = 0, 1

p = C.c_void_p
i64 = C.c_int64
i32 = C.c_int
f32 = C.c_float
fp = C.c_void_p  # device pointers are passed as integers / void*


class BlockConfig(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "batch", "seq", "dim", "heads", "head_dim", "hidden", "chunk", "attn_k", "mlp_k",
        "head0", "heads_local", "f0", "f_local", "t0", "t_local")]


# name -> (restype, [argtypes])
SIGNATURES = {
    "csd_abi_version": (C.c_int, []),
    "csd_last_error": (C.c_char_p, []),
    "csd_status_name": (C.c_char_p, [i32]),
    "csd_ctx_create": (i32, [C.c_int, C.POINTER(p)]),
    "csd_ctx_destroy": (i32, [p]),
    "csd_ctx_sync": (i32, [p, p]),
    "csd_ctx_launch_count": (i64, [p]),
    "csd_ctx_set_validation": (i32, [p, C.c_int]),
    "csd_ctx_set_sorted_topk": (i32, [p, C.c_int]),
    "csd_ctx_set_lpt": (i32, [p, C.c_int]),
    "csd_device_alloc": (i32, [C.c_size_t, C.POINTER(p)]),
    "csd_device_free": (i32, [p]),
    "csd_copy_to_device": (i32, [p, p, C.c_size_t]),
    "csd_copy_to_host": (i32, [p, p, C.c_size_t]),
    "csd_cast": (i32, [p, fp, fp, i64, C.c_int, p]),
    "csd_mlp_preact": (i32, [p, i32, fp, fp, fp, i64, i64, i64, i64, fp, p]),
    "csd_voxel_permutation": (i32, [i64] * 6 + [p]),
    "csd_voxel_reorder": (i32, [p, fp, fp] + [i64] * 8 + [C.c_int, p]),
    "csd_select_top_k": (i32, [p, fp, i64, i64, i64, fp, fp, p]),
    "csd_validate_index_set": (i32, [p, fp, fp, i64, i64, i64, p]),
    "csd_dense_attention": (i32, [p, i32, i32, fp, fp, fp, i64, i64, i64, i64, fp, p]),
    "csd_column_sum_attention": (i32, [p, i32, i32, fp, fp, fp, fp, fp, i64, i64, i64, i64, i64,
                                       fp, fp, fp, fp, p]),
    "csd_sparse_delta_attention": (i32, [p, i32, i32, fp, fp, fp, fp, fp, i64, i64, fp, f32,
                                         i64, i64, i64, i64, fp, p]),
    "csd_dense_mlp": (i32, [p, i32, fp, fp, fp, fp, fp, i64, i64, i64, i64, i64, fp, fp, p]),
    "csd_mlp_tile_means": (i32, [p, i32, fp, fp, i64, i64, i64, i64, i64, fp, p]),
    "csd_mlp_change_indices": (i32, [p, i32, fp, fp, fp, i64, i64, i64, i64, i64, i64, fp, fp, p]),
    "csd_sparse_delta_mlp": (i32, [p, i32, fp, fp, fp, fp, fp, fp, i64, i64, i64, i64, i64, i64,
                                   fp, fp, p]),
    "csd_mlp_act_cache_to_ref": (i32, [p, i32, fp, i64, i64, i64, i64, fp, p]),
    "csd_project": (i32, [p, i32, fp, fp, i64, i64, i64, i64, fp, p]),
    "csd_add": (i32, [p, i32, fp, fp, i64, fp, p]),
    "csd_block_create": (i32, [p, i32, C.POINTER(BlockConfig)] + [fp] * 8 + [C.POINTER(p)]),
    "csd_block_destroy": (i32, [p]),
    "csd_block_reset": (i32, [p]),
    "csd_block_cache_arena": (i32, [p, C.POINTER(p), C.POINTER(C.c_size_t)]),
    "csd_block_bind_cache_arena": (i32, [p, p, C.c_size_t]),
    "csd_block_step": (i32, [p, fp, fp, C.c_int, fp, fp, i64, p]),
    "csd_block_cache": (i32, [p, C.c_int, fp, fp, p]),
    "csd_block_attn_partial": (i32, [p, fp, C.c_int, fp, p]),
    "csd_block_attn_heads": (i32, [p, fp, C.c_int, fp, p]),
    "csd_block_rows_step": (i32, [p, fp, fp, i64, C.c_int, fp, p]),
    "csd_block_mlp_dense_partial": (i32, [p, fp, fp, p]),
    "csd_block_mlp_candidates": (i32, [p, fp, fp, fp, p]),
    "csd_block_mlp_sparse_partial": (i32, [p, fp, fp, fp, i64, fp, p]),
    "csd_residual_add": (i32, [p, fp, fp, i64, fp, p]),
    "csd_resolve_schedule": (i32, [i64, i64, C.c_int, i64, i64, C.POINTER(C.c_int32)]),
    "csd_latent_axpy": (i32, [p, i32, fp, f32, fp, i64, fp, p]),
    "csd_r_squared": (i32, [p, fp, fp, fp, i64, C.POINTER(C.c_double), p]),
    "csd_index_set_to_masks": (i32, [p, fp, fp, i64, i64, i64, fp, p]),
}


def header_symbols() -> list[str]:
    """Every function the public header declares (tests check the .so exports them)."""
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(csd_[a-z0-9_]+)\s*\(", text)))


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run `python -m paper_2506_03275_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
