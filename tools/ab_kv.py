"""cfg2 key/value (2^28 records, payload = index): step, per-pass device
times and a full stability check.  A/B runs of the KV passes (environment
switches are read once per process)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import paper_2107_01391_b200 as rs  # noqa: E402
from ab_partition import profile  # noqa: E402
from oracle import Oracle  # noqa: E402


def main():
    lib = rs._lib.load()
    n = 1 << 28
    k = torch.empty(n, dtype=torch.int32, device="cuda")
    rs._check(lib.rs_gen_u32(Oracle().config_seed(2), 0, n, 10**6, rs._ptr(k), rs._stream()))
    v = torch.empty_like(k)
    rs._check(lib.rs_gen_iota_u32(0, n, rs._ptr(v), rs._stream()))
    res = {"env": {x: os.environ[x] for x in os.environ if x.startswith("RSB_")}}
    res["kv"] = profile(lambda: rs.sort_u32_kv(k, v, key_digits=6), steps=10)
    ko, vo, rep = rs.sort_u32_kv(k, v, key_digits=6)
    same = ko[1:] == ko[:-1]
    res["ok"] = bool((ko[1:] >= ko[:-1]).all()) and bool((vo[1:][same] > vo[:-1][same]).all()) and \
        bool(torch.equal(k[vo.long()], ko))
    res["report"] = [rep.written, rep.cells_traversed, rep.spec.total_digits]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
