"""ctypes binding of the C-ABI in include/recsort_b200.h.

Loads the in-tree ``librecsort_b200.so`` (built by ``__graft_entry__.build()``
or ``python -m paper_2107_01391_b200.build``).  There is no fallback: if the
library is missing, importing the sort API raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_int, c_uint32, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RS_LIB_PATH") or os.path.join(HERE, "librecsort_b200.so")  # override: A/B timing only

# rs_status, in recsort::errc order + 1 (proj/include/recsort/error.hpp:10-23)
STATUS_NAMES = {
    0: "ok",
    1: "parse_error",
    2: "negative_value",
    3: "non_finite",
    4: "cell_budget_exceeded",
    5: "symbol_out_of_alphabet",
    6: "spec_mismatch",
    7: "buffer_too_small",
    8: "range_exceeded",
    9: "out_of_range",
    10: "invalid_range",
    11: "insufficient_data",
    12: "invalid_argument",
    100: "cuda_error",
    101: "nccl_error",
    102: "no_device",
}
RS_OK = 0
RS_BUFFER_TOO_SMALL = 7
DEFAULT_CELL_BUDGET = 100_000_000  # key_model.hpp:16
RS_NUM_PASSES = 13


class RsKeySpec(ctypes.Structure):
    _fields_ = [("radix", c_uint32), ("total_digits", c_uint32), ("integer_digits", c_uint32)]


class RsReport(ctypes.Structure):
    _fields_ = [("written", c_uint64), ("cells_traversed", c_uint64), ("spec", RsKeySpec)]


class RsOptions(ctypes.Structure):
    _fields_ = [("max_cells", c_uint64), ("key_digits", c_uint32), ("msd", c_uint32)]


# (name, restype, argtypes) for every symbol include/recsort_b200.h declares.
SIGNATURES = {
    "rs_last_error": (c_char_p, []),
    "rs_status_name": (c_char_p, [c_int]),
    "rs_version": (c_char_p, []),
    "rs_release_workspaces": (None, []),
    "rs_launch_count": (c_uint64, []),
    "rs_profile_enable": (None, [c_int]),
    "rs_profile_reset": (None, []),
    "rs_profile_read": (c_int, [c_void_p, c_void_p]),
    "rs_pass_name": (c_char_p, [c_int]),
    "rs_sort_u32": (c_int, [c_void_p, c_uint64, c_void_p, c_uint64, POINTER(RsOptions), POINTER(RsReport), c_void_p]),
    "rs_sort_i64": (c_int, [c_void_p, c_uint64, c_void_p, c_uint64, POINTER(RsOptions), POINTER(RsReport), c_void_p]),
    "rs_sort_u32_kv": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p, c_void_p, c_uint64, POINTER(RsOptions), POINTER(RsReport), c_void_p]),
    "rs_sort_u32_multi": (c_int, [c_uint32, POINTER(c_int), POINTER(c_void_p), POINTER(c_uint64), POINTER(c_void_p),
                                  POINTER(c_uint64), POINTER(c_uint64), POINTER(RsOptions), POINTER(RsReport)]),
    "rs_sort_f64": (c_int, [c_void_p, c_uint64, c_uint32, c_void_p, c_uint64, POINTER(RsOptions), POINTER(RsReport), c_void_p]),
    "rs_float_to_decimal": (c_int, [c_void_p, c_uint64, c_uint32, c_void_p, c_void_p]),
    "rs_sort_fixed_str": (c_int, [c_void_p, c_uint64, c_uint32, c_char_p, c_void_p, c_uint64, POINTER(RsOptions), POINTER(RsReport), c_void_p]),
    "rs_sort_keys": (c_int, [c_void_p, c_uint64, RsKeySpec, c_void_p, c_uint64, POINTER(RsOptions), POINTER(RsReport), c_void_p]),
    "rs_sort_decimal_strings": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p, c_uint64, POINTER(RsOptions), POINTER(RsReport), c_void_p]),
    "rs_format_decimals": (c_int, [c_void_p, c_uint64, c_uint32, c_void_p, c_uint64, c_void_p, POINTER(c_uint64), c_void_p]),
    "rs_sort_u32_host": (c_int, [c_void_p, c_uint64, c_void_p, POINTER(RsOptions), POINTER(RsReport), c_void_p]),
    "rs_sort_u32_kv_host": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p, c_void_p, POINTER(RsOptions), POINTER(RsReport), c_void_p]),
    "rs_count_u32": (c_int, [c_void_p, c_uint64, c_void_p, c_uint64, POINTER(c_uint32), c_void_p]),
    "rs_emit_u32": (c_int, [c_void_p, c_uint64, c_uint64, c_uint64, c_uint32, c_void_p, c_uint64, POINTER(c_uint64), c_void_p]),
    "rs_emit_part_u32": (c_int, [c_void_p, c_uint64, c_uint32, c_uint32, c_void_p, c_uint64, POINTER(c_uint64),
                                 POINTER(c_uint64), c_void_p]),
    "rs_bucket_hist_u32": (c_int, [c_void_p, c_uint64, c_uint64, c_void_p, c_uint32, c_void_p]),
    "rs_partition_u32": (c_int, [c_void_p, c_uint64, c_uint64, POINTER(c_uint32), c_uint32, c_void_p, POINTER(c_uint64), c_void_p]),
    "rs_kv_place_u32": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p, c_void_p, c_uint64, POINTER(c_uint64),
                                POINTER(c_uint64), c_uint32, c_void_p]),
    "rs_part_counts_u32": (c_int, [c_void_p, c_uint64, c_uint64, POINTER(c_uint32), c_uint32, POINTER(c_uint64),
                                   c_void_p]),
    "rs_partition_u32_to": (c_int, [c_void_p, c_uint64, c_uint64, POINTER(c_uint32), c_uint32, POINTER(c_uint64),
                                    POINTER(c_uint64), c_void_p]),
    "rs_checked_pow": (c_int, [c_uint64, c_uint32, POINTER(c_uint64)]),
    "rs_make_key_spec": (c_int, [c_uint32, c_uint32, c_uint32, c_uint64, POINTER(RsKeySpec)]),
    "rs_strings_to_keys": (c_int, [c_void_p, c_uint64, c_uint32, c_char_p, c_void_p, POINTER(RsOptions),
                                   POINTER(RsKeySpec), c_void_p]),
    "rs_build_count_space": (c_int, [c_void_p, c_uint64, RsKeySpec, c_uint64, c_void_p, POINTER(c_uint64),
                                     POINTER(ctypes.c_int64), c_void_p]),
    "rs_extract": (c_int, [c_void_p, RsKeySpec, c_uint64, POINTER(c_uint64), POINTER(ctypes.c_int64), c_void_p,
                           c_uint64, POINTER(RsReport), c_void_p]),
    "rs_parse_decimals": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p, c_void_p, c_void_p]),
    "rs_normalize_decimal_strings": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p, POINTER(RsOptions),
                                             POINTER(RsKeySpec), c_void_p]),
    "rs_gen_u32": (c_int, [c_uint64, c_uint64, c_uint64, c_uint64, c_void_p, c_void_p]),
    "rs_gen_iota_u32": (c_int, [c_uint64, c_uint64, c_void_p, c_void_p]),
    "rs_gen_f64_cfg3": (c_int, [c_uint64, c_uint64, c_uint64, c_void_p, c_uint32, c_void_p, c_void_p]),
    "rs_gen_str_cfg4": (c_int, [c_uint64, c_uint64, c_uint64, c_void_p, c_void_p]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the CUDA library (raises if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(there is no CPU implementation of the sort)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def header_symbols(header: str) -> list[str]:
    """Function names declared in include/recsort_b200.h."""
    import re

    text = open(header).read()
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", text)))
