"""B200-native Recombinant Sort hot path (arXiv 2107.01391).

Host-side mirror of the reference's operator interface over the C-ABI in
``include/recsort_b200.h``:

* ``sort_integers`` / ``sort_decimals`` / ``sort_strings`` keep the names,
  arguments, return shape ``(values, ExtractionReport)`` and error behaviour of
  the reference's Python module (proj/python/bindings.cpp:45-72,
  proj/python/recsort/__init__.py) — ``Error`` derives from ``ValueError``.
* ``sort_u32`` / ``sort_u32_kv`` / ``sort_i64`` / ``sort_f64`` /
  ``sort_fixed_str`` / ``sort_keys`` are the device-tensor entry points
  (``recombinant_sort`` dispatches among them), one per C-ABI function.

All sorting runs in the CUDA library; PyTorch only provides device memory
and the current stream.  Without the built library or a GPU the calls raise.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib
from ._lib import DEFAULT_CELL_BUDGET, RsKeySpec, RsOptions, RsReport

__version__ = "0.1.0"

DEFAULT_ALPHABET = "abcdefghijklmnopqrstuvwxyz"


class Error(ValueError):
    """recsort::Error (error.hpp:27-36); ``code`` is the errc name."""

    def __init__(self, code: str, message: str):
        super().__init__(message)
        self.code = code


@dataclass(frozen=True)
class KeySpec:
    radix: int
    total_digits: int
    integer_digits: int

    @property
    def scale(self) -> int:
        return self.total_digits - self.integer_digits


@dataclass(frozen=True)
class ExtractionReport:
    """ExtractionReport (extraction.hpp:12-15) plus the facade's KeySpec."""

    written: int
    cells_traversed: int
    spec: KeySpec

    def __repr__(self) -> str:
        return f"ExtractionReport(written={self.written}, cells_traversed={self.cells_traversed})"


def _check(status: int) -> None:
    if status != _lib.RS_OK:
        lib = _lib.load()
        msg = lib.rs_last_error().decode(errors="replace")
        raise Error(_lib.STATUS_NAMES.get(status, str(status)), msg)


def _report(r: RsReport) -> ExtractionReport:
    return ExtractionReport(int(r.written), int(r.cells_traversed),
                            KeySpec(int(r.spec.radix), int(r.spec.total_digits), int(r.spec.integer_digits)))


def _opts(max_cells: int, key_digits: int = 0, msd: bool = False) -> RsOptions:
    return RsOptions(int(max_cells), int(key_digits), 1 if msd else 0)


def _torch():
    import torch

    return torch


def _stream():
    torch = _torch()
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # skips building a Stream object per call
    if raw is not None:
        return ctypes.c_void_p(raw(torch.cuda.current_device()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None and t.numel() else 0)


def _cuda_tensor(t, dtypes, what):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{what} must be a CUDA tensor")
    if t.dtype not in dtypes:
        raise TypeError(f"{what} must have dtype in {dtypes}, got {t.dtype}")
    return t if t.is_contiguous() else t.contiguous()


# ----------------------------------------------------------- device API
def sort_u32(keys, *, max_cells: int = DEFAULT_CELL_BUDGET, key_digits: int = 0, out=None, msd: bool = False):
    """sort_integers for uint32 keys held in an int32/uint32 CUDA tensor.

    Returns ``(sorted, report)``; ``sorted`` has the input's dtype.  With
    ``msd=True`` a key space above ``max_cells`` is split by MSD bucket passes
    instead of raising cell_budget_exceeded."""
    torch = _torch()
    keys = _cuda_tensor(keys, (torch.int32, torch.uint32), "keys")
    n = keys.numel()
    if out is None:
        out = torch.empty_like(keys)
    rep = RsReport()
    lib = _lib.load()
    _check(lib.rs_sort_u32(_ptr(keys), n, _ptr(out), out.numel(),
                           ctypes.byref(_opts(max_cells, key_digits, msd)), ctypes.byref(rep), _stream()))
    return out, _report(rep)


def sort_u32_multi(shards, *, max_cells: int = DEFAULT_CELL_BUDGET):
    """sort_integers over uint32 keys spread across CUDA tensors on one or
    more devices (rs_sort_u32_multi): returns (outputs, report), output g on
    shard g's device holding slice g of the sorted whole (contiguous cell
    ranges of about total/len(shards) keys)."""
    torch = _torch()
    shards = [_cuda_tensor(s, (torch.int32, torch.uint32), "shard") for s in shards]
    g = len(shards)
    total = sum(s.numel() for s in shards)
    outs = [torch.empty(max(total, 1), dtype=s.dtype, device=s.device) for s in shards]
    devs = (ctypes.c_int * g)(*[s.device.index for s in shards])
    keys = (ctypes.c_void_p * g)(*[s.data_ptr() for s in shards])
    ns = (ctypes.c_uint64 * g)(*[s.numel() for s in shards])
    outp = (ctypes.c_void_p * g)(*[o.data_ptr() for o in outs])
    caps = (ctypes.c_uint64 * g)(*[o.numel() for o in outs])
    written = (ctypes.c_uint64 * g)()
    rep = RsReport()
    torch.cuda.synchronize()
    _check(_lib.load().rs_sort_u32_multi(g, devs, keys, ns, outp, caps, written, ctypes.byref(_opts(max_cells)),
                                         ctypes.byref(rep)))
    return [o[: int(w)] for o, w in zip(outs, written)], _report(rep)


def sort_u32_kv(keys, vals, *, max_cells: int = DEFAULT_CELL_BUDGET, key_digits: int = 0):
    """Stable key/value sort (uint32 keys, uint32 payloads)."""
    torch = _torch()
    keys = _cuda_tensor(keys, (torch.int32, torch.uint32), "keys")
    vals = _cuda_tensor(vals, (torch.int32, torch.uint32), "vals")
    if vals.numel() != keys.numel():
        raise ValueError("keys and vals differ in length")
    ko, vo = torch.empty_like(keys), torch.empty_like(vals)
    rep = RsReport()
    _check(_lib.load().rs_sort_u32_kv(_ptr(keys), _ptr(vals), keys.numel(), _ptr(ko), _ptr(vo), ko.numel(),
                                      ctypes.byref(_opts(max_cells, key_digits)), ctypes.byref(rep), _stream()))
    return ko, vo, _report(rep)


def sort_i64(values, *, max_cells: int = DEFAULT_CELL_BUDGET, key_digits: int = 0, msd: bool = False):
    """sort_integers for non-negative int64 values in a CUDA tensor.  With
    ``msd=True`` a key space above ``max_cells`` is split by MSD bucket passes
    over the values' bit width."""
    torch = _torch()
    values = _cuda_tensor(values, (torch.int64,), "values")
    out = torch.empty_like(values)
    rep = RsReport()
    _check(_lib.load().rs_sort_i64(_ptr(values), values.numel(), _ptr(out), out.numel(),
                                   ctypes.byref(_opts(max_cells, key_digits, msd)), ctypes.byref(rep), _stream()))
    return out, _report(rep)


def sort_f64(x, scale: int, *, max_cells: int = DEFAULT_CELL_BUDGET, key_digits: int = 0):
    """float_to_decimal(x, scale) per element, then the count-grid sort.

    Returns ``(mantissas, report)`` with the sorted uint64 mantissas stored in
    an int64 tensor (DecimalKeySortResult::keys)."""
    torch = _torch()
    x = _cuda_tensor(x, (torch.float64,), "x")
    out = torch.empty(x.numel(), dtype=torch.int64, device=x.device)
    rep = RsReport()
    _check(_lib.load().rs_sort_f64(_ptr(x), x.numel(), int(scale), _ptr(out), out.numel(),
                                   ctypes.byref(_opts(max_cells, key_digits)), ctypes.byref(rep), _stream()))
    return out, _report(rep)


def float_to_decimal_column(x, scale: int):
    """float_to_decimal(x[i], scale).mantissa for a float64 CUDA tensor
    (key_model.cpp:135-158, every double; errors as the reference's for the
    first failing element).  Returns the uint64 mantissas in an int64 tensor."""
    torch = _torch()
    x = _cuda_tensor(x, (torch.float64,), "x")
    out = torch.empty(x.numel(), dtype=torch.int64, device=x.device)
    _check(_lib.load().rs_float_to_decimal(_ptr(x), x.numel(), int(scale), _ptr(out), _stream()))
    return out


def sort_fixed_str(records, *, alphabet: str = DEFAULT_ALPHABET, max_cells: int = DEFAULT_CELL_BUDGET,
                   msd: bool = False):
    """sort_strings over a uint8 CUDA tensor of shape (n, width) of NUL-padded
    records.  ``msd=True`` splits grids above the budget."""
    torch = _torch()
    records = _cuda_tensor(records, (torch.uint8,), "records")
    if records.dim() != 2:
        raise ValueError("records must have shape (n, width)")
    n, width = records.shape
    out = torch.empty_like(records)
    rep = RsReport()
    alpha = alphabet if isinstance(alphabet, bytes) else alphabet.encode()  # bytes: any byte alphabet
    _check(_lib.load().rs_sort_fixed_str(_ptr(records), n, width, alpha, _ptr(out), n,
                                         ctypes.byref(_opts(max_cells, 0, msd)), ctypes.byref(rep), _stream()))
    return out, _report(rep)


def sort_keys(keys, spec: KeySpec, *, max_cells: int = DEFAULT_CELL_BUDGET):
    """sort_keys (extraction.cpp:34-45): uint64 keys of ``spec`` in an int64
    CUDA tensor."""
    torch = _torch()
    keys = _cuda_tensor(keys, (torch.int64,), "keys")
    out = torch.empty_like(keys)
    rep = RsReport()
    _check(_lib.load().rs_sort_keys(_ptr(keys), keys.numel(),
                                    RsKeySpec(spec.radix, spec.total_digits, spec.integer_digits),
                                    _ptr(out), out.numel(), ctypes.byref(_opts(max_cells)), ctypes.byref(rep),
                                    _stream()))
    return out, _report(rep)


def recombinant_sort(data, *args, **kwargs):
    """The recombinant_sort overload set: dispatch on the tensor's dtype."""
    torch = _torch()
    if isinstance(data, tuple):
        return sort_u32_kv(data[0], data[1], *args, **kwargs)
    if data.dtype in (torch.int32, torch.uint32):
        return sort_u32(data, *args, **kwargs)
    if data.dtype == torch.int64:
        return sort_i64(data, *args, **kwargs)
    if data.dtype == torch.float64:
        return sort_f64(data, *args, **kwargs)
    if data.dtype == torch.uint8:
        return sort_fixed_str(data, *args, **kwargs)
    raise TypeError(f"no recombinant_sort overload for {data.dtype}")


# ------------------------------------------- reference Python API mirror
def _device():
    torch = _torch()
    if not torch.cuda.is_available():
        raise Error("no_device", "no CUDA device is visible; recsort_b200 has no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def sort_integers(values, max_cells: int = DEFAULT_CELL_BUDGET):
    """Sort non-negative integers; returns (sorted values, report)
    (bindings.cpp:57-64 -> sort.cpp:29-59)."""
    torch = _torch()
    dev = _device()
    t = torch.tensor(list(values), dtype=torch.int64).to(dev)
    out, rep = sort_i64(t, max_cells=max_cells)
    return out.cpu().tolist(), rep


def _format_scaled(mantissa: int, scale: int) -> str:
    """format_scaled_decimal (key_model.cpp:170-180)."""
    p = 10 ** scale
    out = str(mantissa // p)
    if scale > 0:
        out += "." + str(mantissa % p).rjust(scale, "0")
    return out



def _string_column(values):
    """Arrow-style column: concatenated UTF-8 bytes and n+1 uint64 offsets."""
    import numpy as np

    enc = [v.encode() for v in values]
    lens = np.fromiter((len(e) for e in enc), dtype=np.uint64, count=len(enc))
    offsets = np.zeros(len(enc) + 1, dtype=np.uint64)
    np.cumsum(lens, out=offsets[1:])
    chars = np.frombuffer(b"".join(enc), dtype=np.uint8)
    return chars, offsets


def sort_decimal_column(chars, offsets, *, max_cells: int = DEFAULT_CELL_BUDGET):
    """sort_decimal_keys over a CUDA string column (uint8 chars, int64/uint64
    offsets of n+1 entries): parse + normalize + count + extract on the GPU.
    Returns (uint64 keys at the dataset scale as an int64 tensor, report)."""
    torch = _torch()
    chars = _cuda_tensor(chars, (torch.uint8,), "chars")
    offsets = _cuda_tensor(offsets, (torch.int64,), "offsets")
    n = offsets.numel() - 1
    out = torch.empty(max(n, 1), dtype=torch.int64, device=offsets.device)
    rep = RsReport()
    _check(_lib.load().rs_sort_decimal_strings(_ptr(chars), _ptr(offsets), n, _ptr(out), n,
                                               ctypes.byref(_opts(max_cells)), ctypes.byref(rep), _stream()))
    return out[:n], _report(rep)


def format_decimal_column(keys, scale: int):
    """format_scaled_decimal on the GPU: (uint8 chars, int64 offsets[n+1])."""
    torch = _torch()
    keys = _cuda_tensor(keys, (torch.int64,), "keys")
    n = keys.numel()
    offsets = torch.empty(n + 1, dtype=torch.int64, device=keys.device)
    need = ctypes.c_uint64()
    lib = _lib.load()
    st = lib.rs_format_decimals(_ptr(keys), n, scale, None, 0, _ptr(offsets), ctypes.byref(need), _stream())
    if st not in (0, _lib.RS_BUFFER_TOO_SMALL):
        _check(st)
    chars = torch.empty(max(need.value, 1), dtype=torch.uint8, device=keys.device)
    _check(lib.rs_format_decimals(_ptr(keys), n, scale, _ptr(chars), chars.numel(), _ptr(offsets),
                                  ctypes.byref(need), _stream()))
    return chars[: need.value], offsets


def sort_decimal_keys(values, max_cells: int = DEFAULT_CELL_BUDGET):
    """normalize + hash + extract without rendering (sort.cpp:7-14); the
    numerals are parsed on the GPU (rs_sort_decimal_strings)."""
    torch = _torch()
    chars, offsets = _string_column(values)
    keys, rep = sort_decimal_column(torch.from_numpy(chars.copy()).to(_device()),
                                    torch.from_numpy(offsets.view("int64")).to(_device()), max_cells=max_cells)
    return [int(k) for k in keys.cpu().numpy().view("uint64")], rep


def sort_decimals(values, max_cells: int = DEFAULT_CELL_BUDGET):
    """Sort decimal numerals; returns (sorted padded values, report)
    (bindings.cpp:48-55 -> sort.cpp:16-27): parse, sort and render on the GPU."""
    torch = _torch()
    chars, offsets = _string_column(values)
    keys, rep = sort_decimal_column(torch.from_numpy(chars.copy()).to(_device()),
                                    torch.from_numpy(offsets.view("int64")).to(_device()), max_cells=max_cells)
    out_chars, out_off = format_decimal_column(keys, rep.spec.scale)
    text = bytes(out_chars.cpu().numpy())
    off = out_off.cpu().numpy()
    return [text[off[i]:off[i + 1]].decode() for i in range(len(off) - 1)], rep


def sort_strings(values, alphabet: str = DEFAULT_ALPHABET, max_cells: int = DEFAULT_CELL_BUDGET):
    """Sort strings lexicographically over a fixed alphabet
    (bindings.cpp:66-73 -> sort.cpp:61-77)."""
    torch = _torch()
    if not alphabet:
        raise Error("invalid_argument", "alphabet is empty")
    if len(set(alphabet)) != len(alphabet):
        raise Error("invalid_argument", "duplicate symbol in alphabet")
    enc = [v.encode() for v in values]
    width = max([len(e) for e in enc] + [1])  # key_model.cpp:228-230; the spec check is the library's
    buf = bytearray(len(enc) * width)
    for i, e in enumerate(enc):
        buf[i * width:i * width + len(e)] = e
    recs = torch.frombuffer(buf, dtype=torch.uint8).reshape(len(enc), width) if enc else \
        torch.empty((0, width), dtype=torch.uint8)
    out, rep = sort_fixed_str(recs.to(_device()), alphabet=alphabet, max_cells=max_cells)
    host = out.cpu().numpy()
    return [bytes(r).rstrip(b"\0").decode() for r in host], rep


__all__ = [
    "DEFAULT_CELL_BUDGET", "Error", "ExtractionReport", "KeySpec", "__version__",
    "sort_integers", "sort_decimals", "sort_decimal_keys", "sort_strings", "sort_decimal_column",
    "format_decimal_column", "float_to_decimal_column",
    "sort_u32", "sort_u32_multi", "sort_u32_kv", "sort_i64", "sort_f64", "sort_fixed_str", "sort_keys",
    "recombinant_sort",
]
