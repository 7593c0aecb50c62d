"""Per-pass device times of the cfg2 key-only step (and, with --cfg3, the
cfg3 float64 step), with an exactness check of cfg2.  Used for A/B runs of
partition variants (a build with a temporary switch, read once per process
from RSB_* environment variables; the committed library has none).

    python tools/ab_partition.py [--cfg3 | --only-cfg3] [--i64]
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_01391_b200 as rs  # noqa: E402
from oracle import Oracle  # noqa: E402


def profile(fn, steps=10):
    lib = rs._lib.load()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    lib.rs_profile_enable(1)
    lib.rs_profile_reset()
    for _ in range(steps):
        fn()
    torch.cuda.synchronize()
    ms = (ctypes.c_double * rs._lib.RS_NUM_PASSES)()
    ln = (ctypes.c_uint64 * rs._lib.RS_NUM_PASSES)()
    lib.rs_profile_read(ms, ln)
    lib.rs_profile_enable(0)
    return {"step": round(a.elapsed_time(b) / steps, 4),
            **{lib.rs_pass_name(i).decode(): round(ms[i] / steps, 4) for i in range(rs._lib.RS_NUM_PASSES) if ln[i]}}


def main():
    lib = rs._lib.load()
    o = Oracle()
    n = 1 << 28
    k = torch.empty(n, dtype=torch.int32, device="cuda")
    rs._check(lib.rs_gen_u32(o.config_seed(2), 0, n, 10**6, rs._ptr(k), rs._stream()))
    out = torch.empty_like(k)
    res = {"env": {x: os.environ[x] for x in os.environ if x.startswith("RSB_")}}
    if "--only-cfg3" not in sys.argv:
        res["cfg2"] = profile(lambda: rs.sort_u32(k, out=out, key_digits=6))
        want = torch.bincount(k.long(), minlength=10**6)
        got = torch.bincount(out.long(), minlength=10**6)
        res["cfg2_ok"] = bool(torch.equal(want, got)) and bool((out[1:] >= out[:-1]).all())
    del k, out
    if "--i64" in sys.argv:  # cfg2 keys as int64 through rs_sort_i64 without key_digits (facade_i64)
        k2 = torch.empty(n, dtype=torch.int32, device="cuda")
        rs._check(lib.rs_gen_u32(o.config_seed(2), 0, n, 10**6, rs._ptr(k2), rs._stream()))
        k64 = k2.long()
        del k2
        res["i64"] = profile(lambda: rs.sort_i64(k64))
        o64, _ = rs.sort_i64(k64)
        res["i64_ok"] = bool(torch.equal(o64, torch.sort(k64).values))
        del k64, o64
    if "--cfg3" in sys.argv or "--only-cfg3" in sys.argv:
        cdf = torch.from_numpy(o.zipf_cdf()).cuda()
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        rs._check(lib.rs_gen_f64_cfg3(o.config_seed(3), 0, n, rs._ptr(cdf), cdf.numel(), rs._ptr(x), rs._stream()))
        res["cfg3"] = profile(lambda: rs.sort_f64(x, 3, key_digits=6))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
