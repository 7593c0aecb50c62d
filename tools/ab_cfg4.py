"""cfg4 (2^26 fixed 8-byte strings over 'a'..'z', MSD on one GPU): three
sorts through rs_sort_fixed_str, for an ncu launch list of the last one.

    ncu --metrics gpu__time_duration.sum --csv python tools/ab_cfg4.py
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
    lib = rs._lib.load()
    n4 = 1 << 26
    recs = torch.empty(n4 * 8, dtype=torch.uint8, device="cuda")
    rs._check(lib.rs_gen_str_cfg4(Oracle().config_seed(4), 0, n4, rs._ptr(recs), rs._stream()))
    so = torch.empty_like(recs)
    opts = rs._opts(rs.DEFAULT_CELL_BUDGET, 0, True)
    rep = rs.RsReport()
    for _ in range(3):
        rs._check(lib.rs_sort_fixed_str(rs._ptr(recs), n4, 8, b"abcdefghijklmnopqrstuvwxyz", rs._ptr(so), n4,
                                        ctypes.byref(opts), ctypes.byref(rep), rs._stream()))
    torch.cuda.synchronize()
    print("ok", rep.written, rep.cells_traversed)


if __name__ == "__main__":
    main()
