"""cfg5 (2^31 full-range uint32, MSD on one GPU): step and per-pass device
times, with an exactness check of a slice.  Used for A/B runs of the MSD
engine (environment switches are read once per process)."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_01391_b200 as rs  # noqa: E402
from oracle import Oracle  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ab_partition import profile  # noqa: E402


def main():
    lib = rs._lib.load()
    n = 1 << 31 if "--full" in sys.argv else 1 << 30
    k = torch.empty(n, dtype=torch.int32, device="cuda")
    rs._check(lib.rs_gen_u32(Oracle().config_seed(5), 0, n, 0, rs._ptr(k), rs._stream()))
    out = torch.empty_like(k)
    res = {"env": {x: os.environ[x] for x in os.environ if x.startswith("RSB_")}, "n": n}
    res["cfg5"] = profile(lambda: rs.sort_u32(k, out=out, key_digits=10, msd=True), steps=5)
    sel = k[((k >> 29) & 7) == 3]
    pos = int((((k >> 29) & 7) < 3).sum())
    res["ok"] = bool(torch.equal(out[pos:pos + sel.numel()], torch.sort(sel).values))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
