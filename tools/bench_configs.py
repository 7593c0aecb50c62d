"""Throughput of every BASELINE.json config on one GPU (bench.py keeps the
headline cfg2).  Inputs are generated on the device from the seeded
SplitMix64 streams, already resident in HBM; each config is
timed over K steps with CUDA events after W warm-up steps, with per-pass
device times from the library's own events.

    python tools/bench_configs.py [--steps 5] [--warmup 2] [--only cfg4,dec]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_01391_b200 as rs  # noqa: E402
from oracle import Oracle  # noqa: E402  (seed derivation and the Zipf table only)

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def timed(fn, steps, warmup):
    lib = rs._lib.load()
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = lib.rs_launch_count()
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    launches = (lib.rs_launch_count() - l0) // steps
    lib.rs_profile_enable(1)
    lib.rs_profile_reset()
    for _ in range(steps):
        fn()
    torch.cuda.synchronize()
    ms_arr = (ctypes.c_double * rs._lib.RS_NUM_PASSES)()
    ln_arr = (ctypes.c_uint64 * rs._lib.RS_NUM_PASSES)()
    lib.rs_profile_read(ms_arr, ln_arr)
    lib.rs_profile_enable(0)
    passes = {lib.rs_pass_name(i).decode(): round(ms_arr[i] / steps, 4) for i in range(rs._lib.RS_NUM_PASSES)
              if ln_arr[i]}
    return ms, launches, passes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    lib = rs._lib.load()
    o = Oracle()
    s = rs._stream
    res = {}

    def record(name, n, bpk, ms, launches, passes, extra=None):
        gk = n / (ms / 1e3) / 1e9
        res[name] = {"keys": n, "ms": round(ms, 4), "gkeys_s": round(gk, 2), "algorithmic_B_per_key": bpk,
                     "hbm_frac": round(bpk * n / (ms / 1e3) / 1e9 / PEAK, 4), "gpu_launches": launches,
                     "passes_ms": passes, **(extra or {})}
        print(name, json.dumps(res[name]), flush=True)

    want = lambda c: not args.only or c in args.only.split(",")  # noqa: E731

    if want("cfg1"):
        n = 1 << 20
        k = torch.empty(n, dtype=torch.int32, device="cuda")
        rs._check(lib.rs_gen_u32(o.config_seed(1), 0, n, 1000, rs._ptr(k), s()))
        out = torch.empty_like(k)
        ms, l, p = timed(lambda: rs.sort_u32(k, out=out), args.steps, args.warmup)
        record("cfg1_u32_1000", n, 8, ms, l, p, {"note": "launch-bound (H4); includes the report sync"})
    if want("cfg2"):
        n = 1 << 28
        k = torch.empty(n, dtype=torch.int32, device="cuda")
        rs._check(lib.rs_gen_u32(o.config_seed(2), 0, n, 10**6, rs._ptr(k), s()))
        out = torch.empty_like(k)
        ms, l, p = timed(lambda: rs.sort_u32(k, out=out, key_digits=6), args.steps, args.warmup)
        record("cfg2_u32_1e6_key_only", n, 8, ms, l, p)
        v = torch.empty_like(k)
        rs._check(lib.rs_gen_iota_u32(0, n, rs._ptr(v), s()))
        ms, l, p = timed(lambda: rs.sort_u32_kv(k, v, key_digits=6), args.steps, args.warmup)
        record("cfg2_u32_1e6_key_value", n, 20, ms, l, p)
        del k, v, out
        torch.cuda.empty_cache()
    if want("cfg3"):
        n = 1 << 28
        cdf = torch.from_numpy(o.zipf_cdf()).cuda()
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        rs._check(lib.rs_gen_f64_cfg3(o.config_seed(3), 0, n, rs._ptr(cdf), cdf.numel(), rs._ptr(x), s()))
        ms, l, p = timed(lambda: rs.sort_f64(x, 3, key_digits=6), args.steps, args.warmup)
        record("cfg3_f64_k_over_1000_zipf", n, 16, ms, l, p)
        del x
        torch.cuda.empty_cache()
    if want("cfg4"):
        n = 1 << 26
        r = torch.empty((n, 8), dtype=torch.uint8, device="cuda")
        rs._check(lib.rs_gen_str_cfg4(o.config_seed(4), 0, n, rs._ptr(r), s()))
        ms, l, p = timed(lambda: rs.sort_fixed_str(r, msd=True), args.steps, args.warmup)
        record("cfg4_str8_msd", n, 40, ms, l, p)
        del r
        torch.cuda.empty_cache()
    if want("cfg5"):
        n = 1 << 31
        k = torch.empty(n, dtype=torch.int32, device="cuda")
        rs._check(lib.rs_gen_u32(o.config_seed(5), 0, n, 0, rs._ptr(k), s()))
        out = torch.empty_like(k)
        ms, l, p = timed(lambda: rs.sort_u32(k, out=out, msd=True, key_digits=10), args.steps, args.warmup)
        record("cfg5_u32_full_msd_1gpu", n, 20, ms, l, p, {"note": "declared 10-digit domain (full uint32)"})
    if want("dec"):
        # cfg3's values as decimal text ("k/1000" rendered with 3
        # fractional digits by rs_format_decimals), parsed + sorted + rendered on the GPU
        n = 1 << 28
        k32 = torch.empty(n, dtype=torch.int32, device="cuda")
        rs._check(lib.rs_gen_u32(o.config_seed(3), 0, n, 10**6, rs._ptr(k32), s()))
        keys = (k32.to(torch.int64) & 0xFFFFFFFF).contiguous()
        del k32
        chars, offsets = rs.format_decimal_column(keys, 3)
        nbytes = chars.numel()
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        rep = rs.RsReport()
        opts = rs._opts(10**9)

        def parse_sort():
            rs._check(lib.rs_sort_decimal_strings(rs._ptr(chars), rs._ptr(offsets), n, rs._ptr(out), n,
                                                  ctypes.byref(opts), ctypes.byref(rep), s()))
        ms, l, p = timed(parse_sort, args.steps, args.warmup)
        record("dec_cfg3_text_parse_sort", n, nbytes / n + 8 + 8, ms, l, p,
               {"text_bytes": nbytes, "note": "numerals k/1000 as text; R chars+offsets, W keys"})
        need = ctypes.c_uint64()
        oc = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")

        def render():
            rs._check(lib.rs_format_decimals(rs._ptr(out), n, 3, rs._ptr(oc), nbytes, rs._ptr(oo),
                                             ctypes.byref(need), s()))
        ms, l, p = timed(render, args.steps, args.warmup)
        record("dec_cfg3_render", n, 8 + nbytes / n + 8, ms, l, p, {"note": "R keys, W chars+offsets"})
        del chars, offsets, out, oc, oo, keys
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
