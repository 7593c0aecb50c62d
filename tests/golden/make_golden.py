"""Generate tests/golden/ref_vectors.npz from the UNMODIFIED reference library.

Run in the container that has /root/reference (the library is compiled from
its sources by oracle/Makefile into oracle/_ref/librecsort_ref.so):

    python tests/golden/make_golden.py

Every array below is an input or an output of the reference's own public API
(sort_integers, float_to_decimal, sort_decimals-style core, strings_to_keys,
oracle_sort, radix_sort_lsd_by) on seeded SplitMix64 inputs, so the GPU tests
and the oracle restatement are pinned to the reference without needing it at
run time.
"""
from __future__ import annotations

import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Oracle, Reference  # noqa: E402


def main() -> None:
    orc, ref = Oracle(), Reference()
    out = {}

    # cfg1 shape (keys in [0,1000)), 4096 keys from the cfg1 stream
    seed1 = orc.config_seed(1)
    k1 = orc.gen_u32(seed1, 0, 4096, 1000)
    s1, r1 = ref.sort_integers(k1.astype(np.int64))
    out["cfg1_keys"], out["cfg1_sorted"] = k1, s1.astype(np.uint32)
    out["cfg1_report"] = np.array([r1[0], r1[1], *r1[2]], dtype=np.uint64)

    # cfg2 shape (keys in [0,10^6)), 20000 keys
    seed2 = orc.config_seed(2)
    k2 = orc.gen_u32(seed2, 0, 20000, 10**6)
    s2, r2 = ref.sort_integers(k2.astype(np.int64))
    out["cfg2_keys"], out["cfg2_sorted"] = k2, s2.astype(np.uint32)
    out["cfg2_report"] = np.array([r2[0], r2[1], *r2[2]], dtype=np.uint64)

    # stable key/value: many collisions (keys in [0,50)), payload = index
    kk = orc.gen_u32(orc.mix(seed2, 7), 0, 4000, 50)
    vv = np.arange(4000, dtype=np.uint32)
    ko, vo = ref.radix_sort_lsd_kv(kk, vv)
    out["kv_keys"], out["kv_vals"], out["kv_sorted_keys"], out["kv_sorted_vals"] = kk, vv, ko, vo

    # float_to_decimal: cfg3 values, near-half-way values, and random doubles
    cdf = orc.zipf_cdf(10**6, 1.2)
    seed3 = orc.config_seed(3)
    x3 = orc.gen_f64_cfg3(seed3, 0, 4096, cdf)
    s3, r3 = ref.sort_f64(x3, 3)
    out["cfg3_x"], out["cfg3_sorted"] = x3, s3
    out["cfg3_report"] = np.array([r3[0], r3[1], *r3[2]], dtype=np.uint64)
    rng = np.random.default_rng(20260101)
    ks = rng.integers(0, 10**7, 3000)
    tricky = [k / 10**s + d for k in ks[:1000] for s in (3,) for d in (0.0,)]
    halfs = [(2 * k + 1) / 2000.0 for k in ks[1000:2000]]            # x.xxx5 at scale 3
    nudged = [np.nextafter((2 * k + 1) / 2000.0, np.inf if k % 2 else -np.inf) for k in ks[2000:]]
    rnd = list(rng.random(2000) * 1000.0) + list(rng.random(1000) * 10.0)
    xs = np.array(tricky + halfs + nudged + rnd + [0.0, 2.345, 0.285, 2.344, 4.5, 7.0], dtype=np.float64)
    for scale in (0, 1, 2, 3, 4, 6):
        ms = np.array([ref.float_to_decimal_status(float(x), scale)[1] for x in xs], dtype=np.uint64)
        out[f"f2d_scale{scale}"] = ms
    out["f2d_x"] = xs

    # strings: 600 random strings of length 0..5 over 'abc' (NUL padded to 5)
    recs = np.zeros((600, 5), dtype=np.uint8)
    g = orc.mix(seed1, 11)
    for i in range(600):
        ln = orc.L.or_sm64_at(g, 2 * i) % 6
        for j in range(ln):
            recs[i, j] = ord("abc"[orc.L.or_sm64_at(g, 1000 + 8 * i + j) % 3])
    out["str_recs"] = recs
    out["str_keys"] = ref.strings_to_keys(recs, "abc")
    srt, rs_ = ref.sort_strings(recs, "abc")
    out["str_sorted"] = srt
    out["str_report"] = np.array([rs_[0], rs_[1], *rs_[2]], dtype=np.uint64)
    # cfg4 shape: 8-char a..z strings, ground truth is oracle_sort
    r4 = orc.gen_str_cfg4(orc.config_seed(4), 0, 3000)
    out["cfg4_recs"], out["cfg4_sorted"] = r4, ref.oracle_sort_strings(r4)

    # PRNG known answers (test_bench.cpp:16-22)
    out["splitmix42_first8"] = np.array(ref.splitmix_stream(42, 8), dtype=np.uint64)

    path = os.path.join(ROOT, "tests", "golden", "ref_vectors.npz")
    np.savez_compressed(path, **out)
    print(path, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
