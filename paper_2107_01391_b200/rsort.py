"""rsort-compatible front end over the GPU path.

The reference's CLI (tools/rsort.cpp) and bench harness (bench.hpp:58-121,
bench.cpp:75-334) reach the algorithm through `sort` and `bench`; this module
keeps their flags, outputs and CSV schema and runs the GPU recombinant sort:

    python -m paper_2107_01391_b200.rsort sort --type decimal --report < values.txt
    python -m paper_2107_01391_b200.rsort bench --sizes 1000,100000 --range 1:10 --cd 0,1 --out gpu.csv

`--alg recombinant` is the GPU sort; the CPU baselines (counting, radix,
bucket, oracle) stay in the reference.  Datasets are the reference's
(`generate`: SplitMix64 draws on the cd-place grid, restated here), so a
bench CSV from this module lines up row for row with the reference's, and
the reference's own `rsort analyze` reads it.  The reference's C++ front
ends themselves (bench::run_matrix, the pybind module) reach the GPU by
relinking against include/recsort/*.hpp and this library
(tests/cpp/Makefile.ref); this module is the Python route.
"""
from __future__ import annotations

import argparse
import decimal
import os
import sys
import time

import numpy as np

CSV_HEADER = "algorithm,n_elements,range_lo,range_hi,cd,trial,seconds,extraction_cost"
GAMMA = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


class Failure(Exception):
    """A reference errc with its message (rsort prints `rsort: <msg>`, exits 1;
    rsort.cpp:529-535)."""

    def __init__(self, code: str, message: str):
        super().__init__(message)
        self.code = code


# ------------------------------------------------------------ data
def splitmix64_mix(seed: int, index: int) -> int:
    """splitmix64_mix (splitmix64.hpp): one step from seed + (index + 1) * gamma."""
    z = (seed + (index + 1) * GAMMA) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def _unit_draws(seed: int, n: int) -> np.ndarray:
    """Splitmix64(seed).next_unit() n times, vectorised (uint64 arithmetic wraps)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (np.arange(1, n + 1, dtype=np.uint64) * np.uint64(GAMMA))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def scaled_bounds(lo: float, hi: float, cd: int) -> tuple[int, int]:
    """[lo, hi) on the cd-place mantissa grid (bench.cpp:35-52)."""
    import math

    if not (math.isfinite(lo) and math.isfinite(hi)) or not lo < hi:
        raise Failure("invalid_range", "range bounds must be finite with lo < hi")
    if lo < 0.0:
        raise Failure("invalid_range", "negative ranges are not supported")
    if cd > 18:
        raise Failure("invalid_range", "more than 18 fractional digits")
    p = float(10 ** cd)
    lo_m = math.ceil(lo * p - 1e-9)
    hi_m = math.ceil(hi * p - 1e-9)
    if hi_m <= lo_m:
        raise Failure("invalid_range", f"no representable values in the range at cd={cd}")
    return lo_m, hi_m


def format_scaled_decimal(m: int, cd: int) -> str:
    """key_model.cpp:170-180."""
    if cd == 0:
        return str(m)
    p = 10 ** cd
    return f"{m // p}.{str(m % p).rjust(cd, '0')}"


def generate(n: int, lo: float, hi: float, cd: int, seed: int) -> list[str]:
    """bench::generate (bench.cpp:75-89): n uniform draws on the cd-place grid."""
    lo_m, hi_m = scaled_bounds(lo, hi, cd)
    span = float(hi_m - lo_m)
    off = (_unit_draws(seed, n) * span).astype(np.int64)  # static_cast truncates toward zero
    m = np.minimum(lo_m + off, hi_m - 1)
    if cd == 0:
        return [str(v) for v in m.tolist()]
    p = 10 ** cd
    return [f"{v // p}.{str(v % p).rjust(cd, '0')}" for v in m.tolist()]


def format_double(v: float) -> str:
    """std::to_chars(double) (bench.cpp:24-28): the shorter of the shortest
    round-trip fixed and scientific forms, fixed on a tie."""
    d = decimal.Decimal(repr(float(v))).normalize()
    fixed = format(d, "f")
    sign, digits, exp = d.as_tuple()
    mant = "".join(map(str, digits)).rstrip("0") or "0"
    e10 = len(digits) + exp - 1 if any(digits) else 0
    sci = ("-" if sign else "") + mant[0] + ("." + mant[1:] if len(mant) > 1 else "")
    sci += ("e-" if e10 < 0 else "e+") + str(abs(e10)).rjust(2, "0")
    return fixed if len(fixed) <= len(sci) else sci


def describe(lo: float, hi: float, cd: int) -> dict:
    """bench::describe (bench.cpp:101-122): the case's key geometry."""
    _, hi_m = scaled_bounds(lo, hi, cd)
    ip = len(str((hi_m - 1) // 10 ** cd))
    n = ip + cd
    rep = (10 ** (n - 1) - 1) // 9
    return {"total_digits": n, "integer_digits": ip, "cell_count": 10 ** n,
            "count_dims": "x".join(["10"] * n),
            "h_min_dims": "2" if n == 1 else f"10x{2 * rep}", "h_max_dims": "1" if n == 1 else f"10x{rep}"}


def case_label(lo: float, hi: float, cd: int) -> str:
    return f"({format_double(lo)},{format_double(hi)}) cd={cd}"


# ------------------------------------------------------------ bench
def run_matrix(sizes, cases, trials: int = 3, seed: int = 42, max_cells: int | None = None,
               algorithms=("recombinant",)) -> list[dict]:
    """bench::run_matrix (bench.cpp:144-228) with the GPU recombinant sort:
    case x size x algorithm x trial, one untimed warm-up per cell; the timed
    call is sort_decimal_keys on the host strings (upload, parse, sort and the
    keys back), as the reference times its sort_decimal_keys."""
    from . import DEFAULT_CELL_BUDGET, sort_decimal_keys

    max_cells = max_cells or DEFAULT_CELL_BUDGET
    for a in algorithms:
        if a != "recombinant":
            raise Failure("invalid_argument", f"--alg {a} is a CPU baseline of the reference; "
                                              "this front end runs the GPU recombinant sort")
    records = []
    for ci, (lo, hi, cd) in enumerate(cases):
        g = describe(lo, hi, cd)
        if g["cell_count"] > max_cells:  # case_key_spec: the budget gate before any work
            raise Failure("cell_budget_exceeded",
                          f"key space needs {g['cell_count']} cells, budget is {max_cells}")
        case_seed = splitmix64_mix(seed, ci)
        for si, n in enumerate(sizes):
            ds_seed = splitmix64_mix(case_seed, si)
            data = generate(n, lo, hi, cd, ds_seed)
            for alg in algorithms:
                if trials == 0:
                    continue
                sort_decimal_keys(data, max_cells)  # warm-up, untimed
                for t in range(trials):
                    t0 = time.perf_counter()
                    _, rep = sort_decimal_keys(data, max_cells)
                    dt = time.perf_counter() - t0
                    records.append({"algorithm": alg, "n_elements": n, "range_lo": lo, "range_hi": hi, "cd": cd,
                                    "trial": t, "seconds": dt, "extraction_cost": rep.cells_traversed})
    return records


def emit_csv(records) -> str:
    """bench::emit_csv (bench.cpp:312-334), the reference's schema."""
    out = [CSV_HEADER]
    for r in records:
        cost = "" if r.get("extraction_cost") is None else str(r["extraction_cost"])
        out.append(",".join([r["algorithm"], str(r["n_elements"]), format_double(r["range_lo"]),
                             format_double(r["range_hi"]), str(r["cd"]), str(r["trial"]),
                             format_double(r["seconds"]), cost]))
    return "\n".join(out) + "\n"


def parse_csv(text: str) -> list[dict]:
    """bench::parse_csv (bench.cpp:365-393)."""
    lines = text.split("\n")
    while lines and not lines[-1]:
        lines.pop()
    if not lines or lines[0] != CSV_HEADER:
        raise Failure("parse_error", "missing or malformed CSV header")
    out = []
    for i, line in enumerate(lines[1:], start=2):
        f = line.split(",")
        if len(f) != 8:
            raise Failure("parse_error", f"line {i}: expected 8 fields, got {len(f)}")

        def num(s, kind, name):
            try:
                v = kind(s)
            except ValueError:
                raise Failure("parse_error", f"line {i}: invalid {name} '{s}'") from None
            return v

        out.append({"algorithm": f[0], "n_elements": num(f[1], int, "n_elements"),
                    "range_lo": num(f[2], float, "range_lo"), "range_hi": num(f[3], float, "range_hi"),
                    "cd": num(f[4], int, "cd"), "trial": num(f[5], int, "trial"),
                    "seconds": num(f[6], float, "seconds"),
                    "extraction_cost": num(f[7], int, "extraction_cost") if f[7] else None})
    return out


# ------------------------------------------------------------ sort
def sort_lines(lines: list[str], kind: str = "decimal", alg: str = "recombinant",
               alphabet: str = "abcdefghijklmnopqrstuvwxyz", max_cells: int | None = None,
               raw: bool = False):
    """rsort `sort` (rsort.cpp:147-270) for --alg recombinant on the GPU:
    (output lines, report)."""
    from . import DEFAULT_CELL_BUDGET, sort_decimals, sort_integers, sort_strings

    max_cells = max_cells or DEFAULT_CELL_BUDGET
    if alg not in ("recombinant", "counting", "radix", "bucket", "oracle"):
        raise Failure("invalid_argument", f"unknown algorithm '{alg}'")
    if alg != "recombinant":
        raise Failure("invalid_argument", f"--alg {alg} is a CPU baseline of the reference; "
                                          "this front end runs the GPU recombinant sort")
    if kind == "decimal":
        if raw:
            raise Failure("invalid_argument", "--raw (original spellings) is not provided by the GPU front end")
        out, rep = sort_decimals(lines, max_cells)
        return out, rep
    if kind == "int":
        values = []
        for line in lines:
            if line.startswith("-"):
                raise Failure("negative_value", f"negative values are not supported: '{line}'")
            if not line or not all("0" <= c <= "9" for c in line) or int(line) >= 1 << 63:  # from_chars<int64_t>
                raise Failure("parse_error", f"invalid integer '{line}'")
            values.append(int(line))
        if raw:
            return _raw_int(lines, values, max_cells)
        out, rep = sort_integers(values, max_cells)
        return [str(v) for v in out], rep
    if kind == "string":
        out, rep = sort_strings(lines, alphabet=alphabet, max_cells=max_cells)
        return out, rep
    raise Failure("invalid_argument", f"unknown --type '{kind}'")


def _raw_int(lines, values, max_cells):
    """--raw for integers: original spellings in stable key order
    (originals_by_key, rsort.cpp:133-145) by the GPU's stable key/value sort."""
    import torch

    from . import sort_u32_kv

    if values and (max(values) >= 1 << 32 or len(values) >= 1 << 30):
        raise Failure("invalid_argument", "--raw on the GPU takes keys below 2^32")
    keys = torch.tensor(values, dtype=torch.int64).to(torch.int32).cuda()
    idx = torch.arange(len(values), dtype=torch.int32, device="cuda")
    _, order, rep = sort_u32_kv(keys, idx, max_cells=max(max_cells, 10 ** 10))
    return [lines[i] for i in order.cpu().tolist()], None


# ------------------------------------------------------------ CLI
def _budget(flag: int | None) -> int:
    from . import DEFAULT_CELL_BUDGET

    if flag:
        return flag
    env = os.environ.get("RSORT_MAX_CELLS")
    if env is not None:
        if not env.isdigit() or int(env) == 0:
            raise Failure("invalid_argument", f"RSORT_MAX_CELLS must be a positive integer, got '{env}'")
        return int(env)
    return DEFAULT_CELL_BUDGET


def _parse_list(text: str, what: str) -> list[int]:
    vals = []
    for item in text.split(","):
        if not item.isdigit():
            raise Failure("invalid_argument", f"invalid {what} '{item}'")
        vals.append(int(item))
    if not vals:
        raise Failure("invalid_argument", f"empty {what} list")
    return vals


def _parse_range(text: str) -> tuple[float, float]:
    if ":" not in text:
        raise Failure("invalid_argument", f"range must be lo:hi, got '{text}'")
    a, b = text.split(":", 1)
    try:
        return float(a), float(b)
    except ValueError:
        raise Failure("invalid_argument", f"range must be lo:hi, got '{text}'") from None


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="rsort", description="Recombinant sort on the GPU (rsort-compatible)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("sort", help="sort newline-delimited values from a file or stdin")
    s.add_argument("--alg", "-a", default="recombinant")
    s.add_argument("--type", "-t", default="decimal", dest="kind")
    s.add_argument("--alphabet", default="abcdefghijklmnopqrstuvwxyz")
    s.add_argument("--in", "-i", default="", dest="input")
    s.add_argument("--max-cells", type=int, default=None)
    s.add_argument("--report", action="store_true")
    s.add_argument("--raw", action="store_true")
    b = sub.add_parser("bench", help="run the timing matrix and emit CSV records")
    b.add_argument("--sizes", default="10,100,1000,10000")
    b.add_argument("--range", action="append", default=[], dest="ranges")
    b.add_argument("--cd", default="0,1,2", dest="cds")
    b.add_argument("--algs", default="recombinant")
    b.add_argument("--trials", type=int, default=3)
    b.add_argument("--seed", type=int, default=42)
    b.add_argument("--out", default="")
    b.add_argument("--max-case-digits", type=int, default=3)
    b.add_argument("--max-cells", type=int, default=None)
    args = ap.parse_args(argv)
    try:
        if args.cmd == "sort":
            if args.input in ("", "-"):
                text = sys.stdin.read()
            else:
                try:
                    text = open(args.input).read()
                except OSError:
                    raise Failure("invalid_argument", f"cannot open input file '{args.input}'") from None
            lines = [ln[:-1] if ln.endswith("\r") else ln for ln in text.split("\n")]
            if lines and lines[-1] == "":
                lines.pop()
            out, rep = sort_lines(lines, args.kind, args.alg, args.alphabet, _budget(args.max_cells), args.raw)
            sys.stdout.write("".join(v + "\n" for v in out))
            if args.report:
                if rep is not None:
                    sys.stderr.write(f"written={rep.written} cells_traversed={rep.cells_traversed}\n")
                else:
                    sys.stderr.write("extraction report is only produced by --alg recombinant\n")
            return 0
        sizes = _parse_list(args.sizes, "size")
        cds = _parse_list(args.cds, "cd")
        algs = [a for a in args.algs.split(",") if a]
        if not algs:
            raise Failure("invalid_argument", "empty --algs list")
        cases = []
        for r in args.ranges or ["1:10", "1:100"]:
            lo, hi = _parse_range(r)
            for cd in cds:
                g = describe(lo, hi, cd)
                if g["total_digits"] > args.max_case_digits:
                    sys.stderr.write(f"skipping case {case_label(lo, hi, cd)}: {g['total_digits']} key digits "
                                     f"exceed --max-case-digits {args.max_case_digits}\n")
                    continue
                cases.append((lo, hi, cd))
        if not cases:
            raise Failure("invalid_argument", "no benchmark cases left to run")
        for lo, hi, cd in cases:
            g = describe(lo, hi, cd)
            print(f"case {case_label(lo, hi, cd)}: count array {g['count_dims']}, H_Min {g['h_min_dims']}, "
                  f"H_Max {g['h_max_dims']}")
        records = run_matrix(sizes, cases, args.trials, args.seed, _budget(args.max_cells), algs)
        if args.out:
            with open(args.out, "w") as f:
                f.write(emit_csv(records))
        for alg in algs:
            print(f"\n{alg} mean seconds")
            print("n_elements" + "".join(f"\t{case_label(*c)}" for c in cases))
            for size in sizes:
                cells = []
                for c in cases:
                    ts = [r["seconds"] for r in records if r["algorithm"] == alg and r["n_elements"] == size
                          and (r["range_lo"], r["range_hi"], r["cd"]) == c]
                    cells.append(f"{sum(ts) / len(ts):.5f}" if ts else "-")
                print(str(size) + "".join(f"\t{x}" for x in cells))
        return 0
    except Failure as e:
        sys.stderr.write(f"rsort: {e}\n")
        return 1
    except Exception as e:  # noqa: BLE001 — the product's Error (a library status) or anything else
        from . import Error

        if isinstance(e, Error):
            sys.stderr.write(f"rsort: {e}\n")
            return 1
        sys.stderr.write(f"rsort: internal error: {e}\n")
        return 2


if __name__ == "__main__":
    sys.exit(main())
