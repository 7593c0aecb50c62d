"""ctypes wrappers over the test oracle.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, as the checker or the CPU
baseline — never by the product package.

* ``Oracle``    — liboracle.so, the C++ restatement in oracle.cpp.
* ``Reference`` — oracle/_ref/librecsort_ref.so, the unmodified reference
  library compiled from /root/reference/proj/src (present only where it was
  built; it travels to the GPU box as a prebuilt file).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_char_p, c_double, c_int, c_uint32, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librecsort_ref.so")
REF_SRC = "/root/reference/proj/src/sort.cpp"


class KeySpecC(ctypes.Structure):
    _fields_ = [("radix", c_uint32), ("total_digits", c_uint32), ("integer_digits", c_uint32)]


class ReportC(ctypes.Structure):
    _fields_ = [("written", c_uint64), ("cells_traversed", c_uint64), ("spec", KeySpecC)]

    def as_tuple(self):
        return (int(self.written), int(self.cells_traversed),
                (int(self.spec.radix), int(self.spec.total_digits), int(self.spec.integer_digits)))


class RefReportC(ctypes.Structure):
    _fields_ = [("written", c_uint64), ("cells_traversed", c_uint64), ("radix", c_uint32),
                ("total_digits", c_uint32), ("integer_digits", c_uint32)]

    def as_tuple(self):
        return (int(self.written), int(self.cells_traversed),
                (int(self.radix), int(self.total_digits), int(self.integer_digits)))


def _p(a: np.ndarray) -> c_void_p:
    return c_void_p(a.ctypes.data if a.size else 0)


def ensure_built() -> None:
    if not os.path.exists(ORACLE_SO) or (os.path.exists(REF_SRC) and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


class OracleError(Exception):
    def __init__(self, status: int):
        super().__init__(f"oracle status {status}")
        self.status = status


class Oracle:
    def __init__(self):
        ensure_built()
        L = ctypes.CDLL(ORACLE_SO)
        self.L = L
        L.or_sm64_next.restype = c_uint64
        L.or_sm64_next.argtypes = [POINTER(c_uint64)]
        L.or_sm64_next_unit.restype = c_double
        L.or_sm64_next_unit.argtypes = [POINTER(c_uint64)]
        L.or_sm64_mix.restype = c_uint64
        L.or_sm64_mix.argtypes = [c_uint64, c_uint64]
        L.or_sm64_at.restype = c_uint64
        L.or_sm64_at.argtypes = [c_uint64, c_uint64]
        L.or_config_seed.restype = c_uint64
        L.or_config_seed.argtypes = [c_uint32]
        L.or_decimal_digit_count.restype = c_uint32
        L.or_decimal_digit_count.argtypes = [c_uint64]
        L.or_float_to_decimal.argtypes = [c_double, c_uint32, POINTER(c_uint64)]
        L.or_sort_keys.argtypes = [c_void_p, c_uint64, KeySpecC, c_uint64, c_void_p, c_uint64, POINTER(ReportC)]
        L.or_sort_integers_i64.argtypes = [c_void_p, c_uint64, c_uint64, c_void_p, POINTER(ReportC)]
        L.or_sort_integers_u32.argtypes = [c_void_p, c_uint64, c_uint64, c_void_p, POINTER(ReportC)]
        L.or_sort_f64.argtypes = [c_void_p, c_uint64, c_uint32, c_uint64, c_void_p, POINTER(ReportC)]
        L.or_strings_to_keys.argtypes = [c_void_p, c_uint64, c_uint32, c_char_p, c_uint64, c_void_p,
                                         POINTER(KeySpecC)]
        L.or_sort_fixed_strings.argtypes = [c_void_p, c_uint64, c_uint32, c_char_p, c_void_p, POINTER(ReportC)]
        L.or_radix_sort_lsd_kv_u32.argtypes = [c_void_p, c_void_p, c_uint64, c_void_p, c_void_p]
        L.or_report_from_sorted.argtypes = [c_void_p, c_uint64, c_uint32, c_uint32, POINTER(ReportC)]
        L.or_gen_u32_mod.argtypes = [c_uint64, c_uint64, c_uint64, c_uint64, c_void_p]
        L.or_zipf_cdf.argtypes = [c_uint32, c_double, c_void_p]
        L.or_gen_f64_cfg3.argtypes = [c_uint64, c_uint64, c_uint64, c_void_p, c_uint32, c_void_p]
        L.or_gen_str_cfg4.argtypes = [c_uint64, c_uint64, c_uint64, c_void_p]

    @staticmethod
    def _ok(st: int) -> None:
        if st != 0:
            raise OracleError(st)

    # PRNG
    def splitmix_stream(self, seed: int, count: int) -> list[int]:
        s = c_uint64(seed)
        return [self.L.or_sm64_next(ctypes.byref(s)) for _ in range(count)]

    def next_unit(self, seed: int) -> float:
        s = c_uint64(seed)
        return self.L.or_sm64_next_unit(ctypes.byref(s))

    def mix(self, seed: int, index: int) -> int:
        return self.L.or_sm64_mix(seed, index)

    def config_seed(self, cfg: int) -> int:
        return self.L.or_config_seed(cfg)

    # key model
    def float_to_decimal(self, x: float, scale: int) -> int:
        m = c_uint64()
        self._ok(self.L.or_float_to_decimal(x, scale, ctypes.byref(m)))
        return m.value

    def float_to_decimal_status(self, x: float, scale: int) -> tuple[int, int]:
        m = c_uint64()
        st = self.L.or_float_to_decimal(x, scale, ctypes.byref(m))
        return st, m.value

    # cycles + facades
    def sort_keys(self, keys: np.ndarray, spec: tuple[int, int, int], max_cells: int = 10**8):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        out = np.empty_like(keys)
        rep = ReportC()
        self._ok(self.L.or_sort_keys(_p(keys), keys.size, KeySpecC(*spec), max_cells, _p(out), out.size,
                                     ctypes.byref(rep)))
        return out, rep.as_tuple()

    def sort_integers_u32(self, keys: np.ndarray, max_cells: int = 10**8):
        keys = np.ascontiguousarray(keys, dtype=np.uint32)
        out = np.empty_like(keys)
        rep = ReportC()
        self._ok(self.L.or_sort_integers_u32(_p(keys), keys.size, max_cells, _p(out), ctypes.byref(rep)))
        return out, rep.as_tuple()

    def sort_integers_i64(self, values: np.ndarray, max_cells: int = 10**8):
        values = np.ascontiguousarray(values, dtype=np.int64)
        out = np.empty_like(values)
        rep = ReportC()
        self._ok(self.L.or_sort_integers_i64(_p(values), values.size, max_cells, _p(out), ctypes.byref(rep)))
        return out, rep.as_tuple()

    def sort_f64(self, x: np.ndarray, scale: int, max_cells: int = 10**8):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(x.size, dtype=np.uint64)
        rep = ReportC()
        self._ok(self.L.or_sort_f64(_p(x), x.size, scale, max_cells, _p(out), ctypes.byref(rep)))
        return out, rep.as_tuple()

    def strings_to_keys(self, recs: np.ndarray, alphabet: str = "abcdefghijklmnopqrstuvwxyz",
                        max_cells: int = 10**8):
        recs = np.ascontiguousarray(recs, dtype=np.uint8)
        n, width = recs.shape
        keys = np.empty(n, dtype=np.uint64)
        spec = KeySpecC()
        self._ok(self.L.or_strings_to_keys(_p(recs), n, width, alphabet.encode(), max_cells, _p(keys),
                                           ctypes.byref(spec)))
        return keys, (spec.radix, spec.total_digits, spec.integer_digits)

    def sort_fixed_strings(self, recs: np.ndarray, alphabet: str = "abcdefghijklmnopqrstuvwxyz"):
        recs = np.ascontiguousarray(recs, dtype=np.uint8)
        n, width = recs.shape
        out = np.empty_like(recs)
        rep = ReportC()
        self._ok(self.L.or_sort_fixed_strings(_p(recs), n, width, alphabet.encode(), _p(out), ctypes.byref(rep)))
        return out, rep.as_tuple()

    def radix_sort_lsd_kv(self, keys: np.ndarray, vals: np.ndarray):
        keys = np.ascontiguousarray(keys, dtype=np.uint32)
        vals = np.ascontiguousarray(vals, dtype=np.uint32)
        ko, vo = np.empty_like(keys), np.empty_like(vals)
        self._ok(self.L.or_radix_sort_lsd_kv_u32(_p(keys), _p(vals), keys.size, _p(ko), _p(vo)))
        return ko, vo

    def report_from_sorted(self, sorted_keys: np.ndarray, radix: int, digits: int):
        s = np.ascontiguousarray(sorted_keys, dtype=np.uint64)
        rep = ReportC()
        self._ok(self.L.or_report_from_sorted(_p(s), s.size, radix, digits, ctypes.byref(rep)))
        return rep.as_tuple()

    # generators
    def gen_u32(self, seed: int, first: int, n: int, bound: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint32)
        self.L.or_gen_u32_mod(seed, first, n, bound, _p(out))
        return out

    def zipf_cdf(self, ranks: int = 10**6, s: float = 1.2) -> np.ndarray:
        cdf = np.empty(ranks, dtype=np.float64)
        self.L.or_zipf_cdf(ranks, s, _p(cdf))
        return cdf

    def gen_f64_cfg3(self, seed: int, first: int, n: int, cdf: np.ndarray) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self.L.or_gen_f64_cfg3(seed, first, n, _p(cdf), cdf.size, _p(out))
        return out

    def gen_str_cfg4(self, seed: int, first: int, n: int) -> np.ndarray:
        out = np.empty((n, 8), dtype=np.uint8)
        self.L.or_gen_str_cfg4(seed, first, n, _p(out))
        return out


class Reference:
    """The unmodified reference library (oracle/_ref), if it was built."""

    @staticmethod
    def available() -> bool:
        if not os.path.exists(REF_SO) and os.path.exists(REF_SRC):
            ensure_built()
        return os.path.exists(REF_SO)

    def __init__(self):
        if not self.available():
            raise FileNotFoundError(REF_SO)
        L = ctypes.CDLL(REF_SO)
        self.L = L
        L.ref_last_error.restype = c_char_p
        L.ref_sort_integers.argtypes = [c_void_p, c_uint64, c_uint64, c_void_p, POINTER(RefReportC)]
        L.ref_sort_keys_core.argtypes = [c_void_p, c_uint64, c_uint32, c_uint32, c_uint32, c_uint64, c_void_p,
                                         POINTER(RefReportC)]
        L.ref_float_to_decimal.argtypes = [c_double, c_uint32, POINTER(c_uint64)]
        L.ref_float_to_decimal_many.argtypes = [c_void_p, c_uint64, c_uint32, c_void_p, c_void_p]
        L.ref_sort_f64.argtypes = [c_void_p, c_uint64, c_uint32, c_uint64, c_void_p, POINTER(RefReportC)]
        L.ref_sort_decimals.argtypes = [c_char_p, c_uint64, c_uint64, c_void_p, c_uint64, POINTER(RefReportC)]
        L.ref_sort_strings.argtypes = [c_void_p, c_uint64, c_uint32, c_char_p, c_uint64, c_void_p,
                                       POINTER(RefReportC)]
        L.ref_strings_to_keys.argtypes = [c_void_p, c_uint64, c_uint32, c_char_p, c_uint64, c_void_p]
        L.ref_oracle_sort_strings.argtypes = [c_void_p, c_uint64, c_uint32, c_void_p]
        L.ref_radix_sort_lsd_kv.argtypes = [c_void_p, c_void_p, c_uint64, c_void_p, c_void_p]
        L.ref_radix_sort_lsd.argtypes = [c_void_p, c_uint64, c_void_p]
        L.ref_splitmix64_next.restype = c_uint64
        L.ref_splitmix64_next.argtypes = [POINTER(c_uint64)]
        L.ref_splitmix64_mix.restype = c_uint64
        L.ref_splitmix64_mix.argtypes = [c_uint64, c_uint64]

    def _ok(self, st: int) -> None:
        if st != 0:
            err = OracleError(st)
            err.message = self.L.ref_last_error().decode(errors="replace")
            raise err

    def sort_integers(self, values: np.ndarray, max_cells: int = 10**8):
        values = np.ascontiguousarray(values, dtype=np.int64)
        out = np.empty_like(values)
        rep = RefReportC()
        self._ok(self.L.ref_sort_integers(_p(values), values.size, max_cells, _p(out), ctypes.byref(rep)))
        return out, rep.as_tuple()

    def sort_keys_core(self, keys: np.ndarray, spec, max_cells: int = 10**8):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        out = np.empty_like(keys)
        rep = RefReportC()
        self._ok(self.L.ref_sort_keys_core(_p(keys), keys.size, spec[0], spec[1], spec[2], max_cells, _p(out),
                                           ctypes.byref(rep)))
        return out, rep.as_tuple()

    def float_to_decimal_status(self, x: float, scale: int) -> tuple[int, int]:
        m = c_uint64()
        st = self.L.ref_float_to_decimal(x, scale, ctypes.byref(m))
        return st, m.value

    def float_to_decimal(self, x: float, scale: int) -> int:
        m = c_uint64()
        self._ok(self.L.ref_float_to_decimal(x, scale, ctypes.byref(m)))
        return m.value

    def float_to_decimal_many(self, x: np.ndarray, scale: int) -> tuple[np.ndarray, np.ndarray]:
        """(mantissas, statuses) of float_to_decimal over every element."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        m = np.empty(x.size, dtype=np.uint64)
        st = np.empty(x.size, dtype=np.int32)
        self.L.ref_float_to_decimal_many(_p(x), x.size, scale, _p(m), _p(st))
        return m, st

    def sort_f64(self, x: np.ndarray, scale: int, max_cells: int = 10**8):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(x.size, dtype=np.uint64)
        rep = RefReportC()
        self._ok(self.L.ref_sort_f64(_p(x), x.size, scale, max_cells, _p(out), ctypes.byref(rep)))
        return out, rep.as_tuple()

    def sort_decimals(self, values: list[str], max_cells: int = 10**8):
        joined = b"".join(v.encode() + b"\0" for v in values)
        cap = len(joined) * 4 + 64
        buf = ctypes.create_string_buffer(cap)
        rep = RefReportC()
        self._ok(self.L.ref_sort_decimals(joined, len(values), max_cells, buf, cap, ctypes.byref(rep)))
        raw = buf.raw.split(b"\0")[: len(values)]
        return [r.decode() for r in raw], rep.as_tuple()

    def sort_strings(self, recs: np.ndarray, alphabet: str = "abcdefghijklmnopqrstuvwxyz",
                     max_cells: int = 10**8):
        recs = np.ascontiguousarray(recs, dtype=np.uint8)
        n, width = recs.shape
        out = np.empty_like(recs)
        rep = RefReportC()
        alpha = alphabet if isinstance(alphabet, bytes) else alphabet.encode()
        self._ok(self.L.ref_sort_strings(_p(recs), n, width, alpha, max_cells, _p(out),
                                         ctypes.byref(rep)))
        return out, rep.as_tuple()

    def strings_to_keys(self, recs: np.ndarray, alphabet: str = "abcdefghijklmnopqrstuvwxyz",
                        max_cells: int = 10**8):
        recs = np.ascontiguousarray(recs, dtype=np.uint8)
        n, width = recs.shape
        keys = np.empty(n, dtype=np.uint64)
        self._ok(self.L.ref_strings_to_keys(_p(recs), n, width, alphabet.encode(), max_cells, _p(keys)))
        return keys

    def oracle_sort_strings(self, recs: np.ndarray):
        recs = np.ascontiguousarray(recs, dtype=np.uint8)
        n, width = recs.shape
        out = np.empty_like(recs)
        self._ok(self.L.ref_oracle_sort_strings(_p(recs), n, width, _p(out)))
        return out

    def radix_sort_lsd_kv(self, keys: np.ndarray, vals: np.ndarray):
        keys = np.ascontiguousarray(keys, dtype=np.uint32)
        vals = np.ascontiguousarray(vals, dtype=np.uint32)
        ko, vo = np.empty_like(keys), np.empty_like(vals)
        self._ok(self.L.ref_radix_sort_lsd_kv(_p(keys), _p(vals), keys.size, _p(ko), _p(vo)))
        return ko, vo

    def radix_sort_lsd(self, values: np.ndarray):
        values = np.ascontiguousarray(values, dtype=np.uint64)
        out = np.empty_like(values)
        self._ok(self.L.ref_radix_sort_lsd(_p(values), values.size, _p(out)))
        return out

    def splitmix_stream(self, seed: int, count: int) -> list[int]:
        s = c_uint64(seed)
        return [self.L.ref_splitmix64_next(ctypes.byref(s)) for _ in range(count)]
