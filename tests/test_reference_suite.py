"""The reference's own C++ tests, acceptance criteria and pybind module,
compiled unmodified from /root/reference against this repository's headers
and linked with the B200 library (tests/cpp/Makefile.ref) — the drop-in
boundary of SURVEY 8(b) proven by the reference's own test code.

Built here (where /root/reference exists, also by __graft_entry__.build());
the binaries travel to the GPU box with the snapshot, where the -m gpu cases
run them.  The CPU cases build and run the host-only test cases."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "cpp", "_ref")
UNIT = os.path.join(OUT, "ref_unit")
ACCEPT = os.path.join(OUT, "ref_acceptance")
REF = "/root/reference/proj"

# Test cases of the reference's unit suite that never reach the device: the
# host objects (new_space, hash_insert, TraverseMaps), the single-key helpers,
# and the reference's own CPU code compiled over our headers (bench harness,
# competitor sorts).
HOST_ONLY = ",".join([
    "new_space*", "hash_insert updates*", "each insertion touches*", "keys from another spec*",
    "digits_of*", "reconstruct_value*", "counting_sort", "radix_sort_lsd", "radix passes*", "bucket_sort",
    "oracle_sort", "all baselines agree*", "splitmix64 reference stream", "generate is*", "generate validates*", "fit_scaling*",
    "the reference cd=1*", "worst_case_constant*", "describe*", "emit_csv*", "csv round-trips*", "parse_csv*",
])
# Acceptance criteria that judge this library (c05, c06 and c08 fit the CPU
# algorithm's timing model: run-time slopes and constants of the host loop;
# c07 is pure arithmetic of the bench helpers and fails in the reference
# itself — proj/test_output.txt:23 — which test_reference_c07_as_recorded pins).
ACCEPTANCE = "c01*,c02*,c03*,c04*,c09*,c10*"


def _build():
    from paper_2107_01391_b200 import build

    build.build()
    if os.path.isdir(REF):
        subprocess.run(["make", "-s", "-f", os.path.join(ROOT, "tests", "cpp", "Makefile.ref"), "-j8"], check=True,
                       cwd=ROOT)


def _need_built():
    if not (os.path.exists(UNIT) and os.path.exists(ACCEPT)):
        pytest.fail("reference suite not built (run __graft_entry__.build() where /root/reference exists)")


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present on this machine")
def test_reference_sources_build_against_our_headers():
    _build()
    assert os.path.exists(UNIT) and os.path.exists(ACCEPT)
    assert any(f.startswith("_core") for f in os.listdir(os.path.join(OUT, "recsort")))


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present on this machine")
def test_reference_host_cases_pass():
    _build()
    r = subprocess.run([UNIT, f"--test-case={HOST_ONLY}"], capture_output=True, text=True, timeout=300)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:]
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_reference_unit_suite_on_gpu():
    _need_built()
    r = subprocess.run([UNIT], capture_output=True, text=True, timeout=900)
    print(r.stdout[-6000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-6000:]


@pytest.mark.gpu
def test_reference_acceptance_on_gpu():
    _need_built()
    r = subprocess.run([ACCEPT, f"--test-case={ACCEPTANCE}"], capture_output=True, text=True, timeout=900)
    print(r.stdout[-6000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-6000:]
    assert r.stdout.count("PASS") >= 6


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present on this machine")
def test_reference_c07_as_recorded():
    """c07 (C = 1 + 10^(d-1)/d below (10d)^2) is host arithmetic of the
    reference's bench helpers and fails in the reference's own run from d=6;
    rebuilt over this library it reports the same line."""
    _build()
    r = subprocess.run([ACCEPT, "--test-case=c07*"], capture_output=True, text=True, timeout=120)
    want = "criterion 07 worst-case constant: FAIL -- C values exact, but C < (10d)^2 fails from d=6 (exact arithmetic)"
    assert want in r.stdout
    assert want in open(os.path.join(REF, "test_output.txt")).read()


SMOKE = r'''
import pytest, recsort
assert recsort._core.__file__.startswith(OUT), recsort._core.__file__
values, report = recsort.sort_decimals(["4.5", "0.3", "2.3", "8.8", "7", "9.2", "4.5", "4.3", "8", "3.2"])
assert values == ["0.3", "2.3", "3.2", "4.3", "4.5", "4.5", "7.0", "8.0", "8.8", "9.2"]
assert (report.written, report.cells_traversed) == (10, 17)
values, report = recsort.sort_integers([3, 1, 2, 2])
assert values == [1, 2, 2, 3] and report.written == 4
assert recsort.sort_strings(["ba", "ab", "aa", "b"])[0] == ["aa", "ab", "b", "ba"]
for call, args, match in [(recsort.sort_decimals, (["-3"],), "negative"), (recsort.sort_decimals, (["123456789012"],), "budget"),
                          (recsort.sort_integers, ([-1],), "")]:
    with pytest.raises(ValueError, match=match):
        call(*args)
assert issubclass(recsort.Error, ValueError)
a = recsort.generate(100, 1, 10, 1, 42)
assert a == recsort.generate(100, 1, 10, 1, 42) and a[0] == "7.6"
c = recsort.worst_case_constant(3)
assert (c.numerator, c.denominator) == (103, 3)
s = recsort.describe(1, 10, 2)
assert (s.count_dims, s.h_min_dims, s.h_max_dims, s.cell_count) == ("10x10x10", "10x22", "10x11", 1000)
print("relinked module OK")
'''


@pytest.mark.gpu
def test_reference_python_module_relinked_on_gpu():
    """The reference's pybind module (proj/python/bindings.cpp), rebuilt over
    this library, through the calls of the reference's python smoke test
    (proj/tests/python/test_smoke.py)."""
    _need_built()
    env = dict(os.environ, PYTHONPATH=OUT)
    code = f"OUT = {OUT!r}\n" + SMOKE
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    print(r.stdout, r.stderr[-3000:])
    assert r.returncode == 0 and "relinked module OK" in r.stdout
