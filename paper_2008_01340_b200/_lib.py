"""ctypes binding of libntt.so (include/ntt.h) -- argument marshalling only.

Every arithmetic step runs in the library's sm_100a kernels; this module only
passes pointers, sizes and scalars.  Loading fails loudly if the library has not
been built (there is no CPU fallback anywhere in the product).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NTT_LIB") or os.path.join(_HERE, "libntt.so")  # NTT_LIB: experiment builds

c_i32, c_i64, c_u64, c_f32, c_f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_double
c_p = ctypes.c_void_p
c_int = ctypes.c_int
c_size = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/ntt.h one to one
SIGNATURES = {
    "ntt_create": (c_int, [ctypes.POINTER(c_p), c_int, c_p]),
    "ntt_destroy": (c_int, [c_p]),
    "ntt_set_stream": (c_int, [c_p, c_p]),
    "ntt_status_string": (ctypes.c_char_p, [c_int]),
    "ntt_last_error": (ctypes.c_char_p, [c_p]),
    "ntt_abi_version": (c_int, []),
    "ntt_launch_count": (c_i64, [c_p]),
    "ntt_fill_uniform": (c_int, [c_p, c_p, c_i64, c_u64, c_u64, c_i64]),
    "ntt_nmf_mu": (c_int, [c_p, c_p, c_i64, c_i64, c_i64, c_i32, c_i32, c_f32, c_p, c_p, c_p]),
    "ntt_decompose_workspace_bytes": (c_size, [c_i32, c_p, c_p]),
    "ntt_decompose": (c_int, [c_p, c_p, c_i32, c_p, c_p, c_i32, c_u64, c_f32, c_p, c_p, c_p, c_size]),
    "ntt_profile_enable": (c_int, [c_p, c_int]),
    "ntt_profile_get": (c_int, [c_p, c_int, ctypes.POINTER(c_i64), ctypes.POINTER(c_f64), ctypes.POINTER(c_f64)]),
    "ntt_profile_get_step": (c_int, [c_p, c_int, c_int, ctypes.POINTER(c_i64), ctypes.POINTER(c_f64),
                                     ctypes.POINTER(c_f64)]),
    "ntt_reconstruct": (c_int, [c_p, c_i32, c_p, c_p, c_p, c_p, c_p, c_p]),
    "ntt_decompose_eps": (c_int, [c_p, c_p, c_i32, c_p, c_f64, c_p, c_i32, c_u64, c_f32, c_p, c_i64, c_p, c_p]),
    "ntt_nmf_bcd": (c_int, [c_p, c_p, c_i64, c_i64, c_i64, c_i32, c_i32, c_f64, c_p, c_p, c_p]),
    "ntt_tt_svd": (c_int, [c_p, c_p, c_i32, c_p, c_f64, c_p, c_p, c_i64, c_p, c_p]),
    "ntt_decompose_bcd": (c_int, [c_p, c_p, c_i32, c_p, c_p, c_i32, c_u64, c_f64, c_p, c_p]),
    "ntt_rank_rule": (c_int, [c_p, c_p, c_i64, c_i64, c_i64, c_f64, ctypes.POINTER(c_i32), c_p]),
    "ntt_generate": (c_int, [c_p, c_i32, c_p, c_p, c_p, c_f32, c_u64, c_u64, c_p]),
    "ntt_compression_ratio": (c_f64, [c_i32, c_p, c_p]),
    "ntt_get_unique_id": (c_int, [c_p]),
    "ntt_create_dist": (c_int, [ctypes.POINTER(c_p), c_int, c_p, c_p, c_int, c_int]),
    "ntt_create_dist_grid": (c_int, [ctypes.POINTER(c_p), c_int, c_p, c_p, c_int, c_int, c_int, c_int]),
    "ntt_dist_grid": (c_int, [c_p, ctypes.POINTER(c_int), ctypes.POINTER(c_int), ctypes.POINTER(c_int),
                              ctypes.POINTER(c_int)]),
    "ntt_dist_rank": (c_int, [c_p]),
    "ntt_dist_size": (c_int, [c_p]),
    "ntt_dist_block": (c_i64, [c_i64, c_int, c_int, ctypes.POINTER(c_i64)]),
    "ntt_debug_persist_trace": (ctypes.POINTER(ctypes.c_uint64), [c_p]),
    "ntt_debug_mu_path": (c_i32, [c_p, c_i64, c_i64, c_i32]),
    "ntt_prefetch_input": (c_int, [c_p, c_p, c_i64]),
    "ntt_debug_bcd_force_correct": (c_int, [c_p, ctypes.c_uint64]),
    "ntt_set_validation": (c_int, [c_p, c_int]),
    "ntt_collective_count": (c_i64, [c_p]),
    "ntt_stream_ceiling": (c_int, [c_p, c_p, c_i64, c_i32, ctypes.POINTER(c_f64)]),
    "ntt_set_dist_exchange": (c_int, [c_p, c_int]),
    "ntt_peer_exchange_count": (c_i64, [c_p]),
    "ntt_debug_fill_uniform_cols": (c_int, [c_p, c_p, c_i32, c_i64, c_i64, c_i64, c_i64, c_i64, c_u64, c_u64]),
    "ntt_debug_gather_last_core": (c_int, [c_p, c_p, c_i64, c_i64, c_i32, c_p]),
}

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2008_01340_b200.build` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
