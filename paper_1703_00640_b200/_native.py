"""ctypes binding of the C ABI in include/truncmul_b200.h.

The shared library is built in-tree (``python -c 'import __graft_entry__ as g;
g.build()'`` or ``make``) as ``paper_1703_00640_b200/libtruncmul_b200.so``.
Importing this module fails loudly when it is missing: there is no CPU
fallback for the product path.
"""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtruncmul_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "truncmul_b200.h")

TMG_OK = 0
TMG_ERR_INPUT_OUT_OF_RANGE = 1
TMG_ERR_NO_VALID_PARAMS = 2
TMG_ERR_UNSUPPORTED_LENGTH = 3
TMG_ERR_PRECISION_FAILURE = 4
TMG_ERR_PLAN_MISMATCH = 5
TMG_ERR_UNSUPPORTED = 6
TMG_ERR_CUDA = 7
TMG_ERR_INTERNAL = 8


class tmg_params(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("b", ctypes.c_int32),
        ("N", ctypes.c_int64),
        ("lam", ctypes.c_int64),
        ("p", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("backend", ctypes.c_int32),
        ("signed_split", ctypes.c_int32),
    ]


class tmg_stats(ctypes.Structure):
    _fields_ = [
        ("max_round_err", ctypes.c_double),
        ("max_abs", ctypes.c_double),
        ("flags", ctypes.c_uint32),
        ("transform_length", ctypes.c_int64),
        ("passes", ctypes.c_int32),
        ("kernels", ctypes.c_int32),
        ("attempts", ctypes.c_int32),
        ("b", ctypes.c_int32),
        ("N", ctypes.c_int64),
        ("first_round_err", ctypes.c_double),
    ]


TMG_STAT_ESCALATED = 1 << 24

# tmg_context_set_option (testing and diagnostics)
TMG_OPT_GENERIC_COLUMN_PASSES = 1
TMG_OPT_FORCE_THREE_PASS = 2
TMG_OPT_GENERIC_ROW_PASS = 3
TMG_OPT_LOOKBACK_CARRY = 4
TMG_OPT_PATCH_SCAN_MAX = 5
TMG_OPT_NO_PDL = 6
TMG_OPT_DEBUG_SYNC = 7
TMG_OPT_NO_GRAPH = 8
TMG_OPT_Z_NATURAL = 9
TMG_OPT_GENERIC_SMALL = 10
TMG_OPT_PREMAP_IN_SPLIT = 11
TMG_OPT_CARRY_KERNELS = 12
TMG_OPT_MAX_ROW = 13
TMG_OPT_SPLIT_AGGREGATES = 14
TMG_OPT_GENERIC_RUNS = 15
TMG_OPT_SPLIT_KERNEL = 16


def header_functions() -> list[str]:
    """Names of every function the C header declares."""
    text = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(tmg_\w+)\s*\(", text, re.M)))


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    i32, i64, u64p, vp = ctypes.c_int32, ctypes.c_int64, P(ctypes.c_uint64), ctypes.c_void_p
    L.tmg_last_error.restype = ctypes.c_char_p
    L.tmg_version.restype = ctypes.c_char_p
    L.tmg_required_precision.argtypes = [i32, i32, i64, P(i32)]
    L.tmg_default_lambda.argtypes = [i32, i32, i32, i32, P(i64)]
    L.tmg_validate_params.argtypes = [P(tmg_params)]
    L.tmg_select_params.argtypes = [i64, i32, i32, i64, i32, P(tmg_params)]
    L.tmg_output_limbs.argtypes = [i32, i64]
    L.tmg_output_limbs.restype = i64
    L.tmg_predicted_sigma.argtypes = [P(tmg_params)]
    L.tmg_predicted_sigma.restype = ctypes.c_double
    L.tmg_context_create.argtypes = [ctypes.c_int, P(vp)]
    L.tmg_context_destroy.argtypes = [vp]
    L.tmg_context_destroy.restype = None
    L.tmg_context_set_stream.argtypes = [vp, vp]
    L.tmg_context_set_escalation.argtypes = [vp, ctypes.c_int]
    L.tmg_synchronize.argtypes = [vp]
    for name in ("tmg_full_product", "tmg_low_product", "tmg_high_product"):
        getattr(L, name).argtypes = [vp, P(tmg_params), u64p, u64p, u64p, P(tmg_stats)]
    L.tmg_product_batched.argtypes = [vp, P(tmg_params), u64p, u64p, i64, u64p,
                                      P(ctypes.c_uint32), P(tmg_stats)]
    L.tmg_cyclic_convolve_f64.argtypes = [vp, i64, P(ctypes.c_double), P(ctypes.c_double),
                                          P(ctypes.c_double)]
    PDbl = P(ctypes.c_double)
    L.tmg_alpha_star_f64.argtypes = [vp, i64, ctypes.c_int32, i64, PDbl, PDbl]
    L.tmg_beta_star_f64.argtypes = [vp, i64, ctypes.c_int32, i64, PDbl, PDbl]
    L.tmg_gamma_dagger_f64.argtypes = [vp, i64, ctypes.c_int32, i64, PDbl, PDbl, PDbl]
    L.tmg_delta_dagger_f64.argtypes = [vp, i64, ctypes.c_int32, i64, PDbl, ctypes.c_double, PDbl]
    for name in ("tmg_split_low_i64", "tmg_split_high_i64"):
        getattr(L, name).argtypes = [vp, P(tmg_params), u64p, P(ctypes.c_int64)]
    L.tmg_product_device.argtypes = [vp, P(tmg_params), vp, vp, vp, i64]
    L.tmg_check.argtypes = [vp, P(tmg_stats)]
    L.tmg_host_alloc.argtypes = [ctypes.c_size_t, P(vp)]
    L.tmg_host_free.argtypes = [vp]
    L.tmg_host_free.restype = None
    L.tmg_device_alloc.argtypes = [ctypes.c_size_t, P(vp)]
    L.tmg_device_free.argtypes = [vp]
    L.tmg_device_free.restype = None
    L.tmg_memcpy_h2d.argtypes = [vp, vp, vp, ctypes.c_size_t]
    L.tmg_memcpy_d2h.argtypes = [vp, vp, vp, ctypes.c_size_t]
    L.tmg_last_kernel_count.argtypes = [vp]
    L.tmg_last_kernel_count.restype = i32
    L.tmg_profile_enable.argtypes = [vp, ctypes.c_int]
    L.tmg_profile_read.argtypes = [vp, ctypes.c_char_p, ctypes.c_int, P(ctypes.c_double),
                                   P(ctypes.c_double), ctypes.c_int, P(ctypes.c_int)]
    L.tmg_debug_read.argtypes = [vp, ctypes.c_int, vp, P(ctypes.c_size_t)]
    L.tmg_context_set_option.argtypes = [vp, i32, i64]
    _lib = L
    return L


def last_error() -> str:
    return load().tmg_last_error().decode(errors="replace")
