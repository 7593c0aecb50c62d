"""One cfg2 key-only sort and one cfg2 key/value sort (2^28 keys), for ncu
captures of individual kernels:

    python tools/profile_one.py [--kv] [--f64] [--cfg4] [--cfg5] [--no-cfg2]
    ncu --set full -k regex:k_outer_scatter -c 1 -o prof python tools/profile_one.py
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_01391_b200 as rs  # noqa: E402
from oracle import Oracle  # noqa: E402


def main():
    n = 1 << 28
    lib = rs._lib.load()
    o = Oracle()
    keys = torch.empty(n, dtype=torch.int32, device="cuda")
    rs._check(lib.rs_gen_u32(o.config_seed(2), 0, n, 10**6, rs._ptr(keys), rs._stream()))
    rep = None
    if "--no-cfg2" not in sys.argv:  # other configs only (their launch lists)
        for _ in range(2):
            out, rep = rs.sort_u32(keys, key_digits=6)
    torch.cuda.synchronize()
    if "--kv" in sys.argv:
        vals = torch.empty_like(keys)
        rs._check(lib.rs_gen_iota_u32(0, n, rs._ptr(vals), rs._stream()))
        for _ in range(2):
            rs.sort_u32_kv(keys, vals, key_digits=6)
    if "--f64" in sys.argv:
        cdf = torch.from_numpy(o.zipf_cdf()).cuda()
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        rs._check(lib.rs_gen_f64_cfg3(o.config_seed(3), 0, n, rs._ptr(cdf), cdf.numel(), rs._ptr(x), rs._stream()))
        for _ in range(2):
            rs.sort_f64(x, 3, key_digits=6)
    if "--cfg4" in sys.argv:
        n4 = 1 << 26
        r4 = torch.empty((n4, 8), dtype=torch.uint8, device="cuda")
        rs._check(lib.rs_gen_str_cfg4(o.config_seed(4), 0, n4, rs._ptr(r4), rs._stream()))
        for _ in range(2):
            rs.sort_fixed_str(r4, msd=True)
        del r4
    if "--cfg5" in sys.argv:
        del keys
        out = None
        torch.cuda.empty_cache()
        n5 = 1 << 31
        k5 = torch.empty(n5, dtype=torch.int32, device="cuda")
        rs._check(lib.rs_gen_u32(o.config_seed(5), 0, n5, 0, rs._ptr(k5), rs._stream()))
        o5 = torch.empty_like(k5)
        rs.sort_u32(k5, out=o5, msd=True)
    torch.cuda.synchronize()
    print("ok", rep)


if __name__ == "__main__":
    main()
