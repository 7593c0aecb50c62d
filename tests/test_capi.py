"""CPU checks of the boundary: the library loads, exports exactly what
include/recsort_b200.h declares, names statuses in errc order, and — with no
GPU — refuses to sort instead of falling back to a CPU path."""
import ctypes
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "recsort_b200.h")
ERRC = ["parse_error", "negative_value", "non_finite", "cell_budget_exceeded", "symbol_out_of_alphabet",
        "spec_mismatch", "buffer_too_small", "range_exceeded", "out_of_range", "invalid_range",
        "insufficient_data", "invalid_argument"]  # error.hpp:10-23


@pytest.fixture(scope="module")
def lib():
    from paper_2107_01391_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        from paper_2107_01391_b200 import build

        build.build()
    return _lib.load()


def test_exports_every_header_symbol(lib):
    from paper_2107_01391_b200 import _lib

    declared = _lib.header_symbols(HEADER)
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert set(declared) == set(_lib.SIGNATURES), "ctypes signatures drifted from the header"


def test_status_names_follow_errc_order(lib):
    for i, name in enumerate(ERRC):
        assert lib.rs_status_name(i + 1).decode() == name
    assert lib.rs_status_name(0).decode() == "ok"
    assert lib.rs_status_name(102).decode() == "no_device"
    assert b"sm_100a" in lib.rs_version()


def test_no_cpu_fallback_without_gpu(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2107_01391_b200._lib import RsOptions, RsReport

    keys = (ctypes.c_uint32 * 4)(3, 1, 2, 2)
    out = (ctypes.c_uint32 * 4)()
    st = lib.rs_sort_u32(ctypes.cast(keys, ctypes.c_void_p), 4, ctypes.cast(out, ctypes.c_void_p), 4,
                         ctypes.byref(RsOptions(0, 0, 0)), ctypes.byref(RsReport()), None)
    assert st == 102
    assert b"no CPU path" in lib.rs_last_error()


def test_python_mirror_raises_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2107_01391_b200 as rs

    with pytest.raises(rs.Error) as e:
        rs.sort_integers([3, 1, 2])
    assert e.value.code == "no_device"
    assert isinstance(e.value, ValueError)  # bindings.cpp:20


def test_format_scaled_helper():
    # format_scaled_decimal (key_model.cpp:170-180), the host rendering the
    # decimal facade's tests compare with
    import paper_2107_01391_b200 as rs

    assert rs._format_scaled(45, 1) == "4.5"
    assert rs._format_scaled(3, 1) == "0.3"
    assert rs._format_scaled(105, 2) == "1.05"
    assert rs._format_scaled(7, 0) == "7"
