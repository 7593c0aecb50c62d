"""The rsort-compatible front end (paper_2107_01391_b200/rsort.py, SURVEY 8f
row 4): the bench datasets, case geometry, CSV schema and number formatting
pinned to the reference's own bench code (oracle/_ref: bench::generate,
describe, emit_csv, case_label), CLI argument errors, and — on a GPU — the
`sort` and `bench` commands against the reference facade."""
import ctypes
import io
import math
import subprocess
import sys

import numpy as np
import pytest

from paper_2107_01391_b200 import rsort


class RefBench:
    def __init__(self, ref):
        L = ref.L
        L.ref_generate.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_double, ctypes.c_uint32,
                                   ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint64]
        L.ref_describe.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_uint32, ctypes.c_char_p,
                                   ctypes.c_uint64]
        L.ref_emit_csv_one.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double, ctypes.c_int,
                                       ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint64]
        self.ref, self.L = ref, L

    def generate(self, n, lo, hi, cd, seed):
        buf = ctypes.create_string_buffer(n * 32 + 16)
        self.ref._ok(self.L.ref_generate(n, lo, hi, cd, seed, buf, len(buf)))
        return buf.raw.split(b"\0")[:n]

    def describe(self, lo, hi, cd):
        buf = ctypes.create_string_buffer(256)
        self.ref._ok(self.L.ref_describe(lo, hi, cd, buf, len(buf)))
        t, i, c, cdims, hmin, hmax = buf.value.decode().split(",")
        return {"total_digits": int(t), "integer_digits": int(i), "cell_count": int(c), "count_dims": cdims,
                "h_min_dims": hmin, "h_max_dims": hmax}

    def emit_one(self, rec):
        buf = ctypes.create_string_buffer(512)
        cost = rec["extraction_cost"]
        self.ref._ok(self.L.ref_emit_csv_one(rec["algorithm"].encode(), rec["n_elements"], rec["range_lo"],
                                             rec["range_hi"], rec["cd"], rec["trial"], rec["seconds"],
                                             cost is not None, cost or 0, buf, len(buf)))
        csv, label = buf.value.decode().split("|")
        return csv, label


@pytest.fixture(scope="module")
def rb(ref):
    return RefBench(ref)


@pytest.mark.parametrize("lo,hi,cd", [(1.0, 10.0, 0), (1.0, 10.0, 2), (1.0, 100.0, 1), (0.0, 1.0, 3),
                                      (2.5, 7.25, 2), (0.0, 1e6, 0), (3.3, 3.31, 4)])
def test_generate_matches_reference(rb, lo, hi, cd):
    for seed in (1, 42, rsort.splitmix64_mix(42, 3), 2**64 - 5):
        want = rb.generate(2000, lo, hi, cd, seed)
        got = rsort.generate(2000, lo, hi, cd, seed)
        assert [g.encode() for g in got] == want


def test_describe_matches_reference(rb):
    for lo, hi, cd in [(1.0, 10.0, 0), (1.0, 10.0, 1), (1.0, 100.0, 1), (0.0, 1.0, 0), (5.0, 99999.0, 2)]:
        assert rsort.describe(lo, hi, cd) == rb.describe(lo, hi, cd)


def test_csv_and_labels_match_reference(rb):
    rng = np.random.default_rng(3)
    vals = [0.0, 1.0, 10.0, 100.0, 0.5, 1e-4, 1.5e-4, 1234567.0, 1e22, 1e21, 123456789012.0, 2.5, 1e-7,
            0.000123, 3.3, 1e15, 1e16, 1e17] + list(10.0 ** rng.uniform(-9, 3, 300))
    for i, s in enumerate(vals):
        rec = {"algorithm": "recombinant", "n_elements": 1000 + i, "range_lo": 1.0 if i % 2 else 0.25,
               "range_hi": 10.0 + i, "cd": i % 3, "trial": i % 4, "seconds": float(s),
               "extraction_cost": None if i % 5 == 0 else 17 * i}
        csv, label = rb.emit_one(rec)
        assert rsort.emit_csv([rec]) == csv
        assert rsort.case_label(rec["range_lo"], rec["range_hi"], rec["cd"]) == label


def test_cli_argument_errors_match_reference_messages():
    err = io.StringIO()
    old = sys.stderr
    sys.stderr = err
    try:
        assert rsort.main(["bench", "--range", "5"]) == 1
        assert rsort.main(["bench", "--sizes", "10,x"]) == 1
        assert rsort.main(["bench", "--range", "1:10", "--cd", "5", "--max-case-digits", "3"]) == 1
    finally:
        sys.stderr = old
    lines = err.getvalue().splitlines()
    assert lines[0] == "rsort: range must be lo:hi, got '5'"
    assert lines[1] == "rsort: invalid size 'x'"
    assert lines[2].startswith("skipping case (1,10) cd=5: 6 key digits exceed --max-case-digits 3")
    assert lines[3] == "rsort: no benchmark cases left to run"


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_cli_sort_decimal_int_string(rs, ref, tmp_path):
    vals = rsort.generate(5000, 1.0, 100.0, 2, 7) + ["0.5", "3"]
    want, wrep = ref.sort_decimals(vals)
    p = tmp_path / "d.txt"
    p.write_text("\n".join(vals) + "\n")
    r = subprocess.run([sys.executable, "-m", "paper_2107_01391_b200.rsort", "sort", "--in", str(p), "--report"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert r.stdout.splitlines() == want
    assert r.stderr.strip() == f"written={wrep[0]} cells_traversed={wrep[1]}"
    ints = [str(v) for v in np.random.default_rng(1).integers(0, 10**5, 3000)]
    out, rep = rsort.sort_lines(ints, "int")
    assert out == [str(v) for v in sorted(map(int, ints))]
    raw, _ = rsort.sort_lines(["007", "7", "3", "07"], "int", raw=True)
    assert raw == ["3", "007", "7", "07"]  # originals, stable by value
    strs = ["bana", "apple", "cher", "app", "b"]  # width 5: 27^5 cells fit the default budget
    out, rep = rsort.sort_lines(strs, "string")
    assert out == sorted(strs)
    r = subprocess.run([sys.executable, "-m", "paper_2107_01391_b200.rsort", "sort", "--type", "int"],
                       input="5\n-3\n", capture_output=True, text=True)
    assert r.returncode == 1 and r.stderr.strip() == "rsort: negative values are not supported: '-3'"


@pytest.mark.gpu
def test_cli_bench_csv(rs, ref, tmp_path):
    """bench --out: the reference schema, one row per (case, size, trial), the
    extraction cost of each row equal to the reference's cells_traversed on
    the same generated dataset."""
    out = tmp_path / "gpu.csv"
    r = subprocess.run([sys.executable, "-m", "paper_2107_01391_b200.rsort", "bench", "--sizes", "100,2000",
                        "--range", "1:10", "--range", "1:100", "--cd", "0,1", "--trials", "2", "--out", str(out)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rows = out.read_text().splitlines()
    assert rows[0] == rsort.CSV_HEADER and len(rows) == 1 + 4 * 2 * 2
    cases = [(1.0, 10.0, 0), (1.0, 10.0, 1), (1.0, 100.0, 0), (1.0, 100.0, 1)]
    for ci, (lo, hi, cd) in enumerate(cases):
        for si, n in enumerate([100, 2000]):
            data = rsort.generate(n, lo, hi, cd, rsort.splitmix64_mix(rsort.splitmix64_mix(42, ci), si))
            _, wrep = ref.sort_decimals(data)
            for t in range(2):
                f = rows[1 + (ci * 2 + si) * 2 + t].split(",")
                assert f[0] == "recombinant" and int(f[1]) == n and int(f[4]) == cd and int(f[5]) == t
                assert int(f[7]) == wrep[1] and math.isfinite(float(f[6]))
    assert "recombinant mean seconds" in r.stdout
