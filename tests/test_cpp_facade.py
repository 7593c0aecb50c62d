"""The drop-in C++ facade (include/recsort/sort.hpp over the C-ABI): the
reference's facade cases restated in tests/cpp/test_facade.cpp.  The build is
checked on CPU; the run needs a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2107_01391_b200")


def _build(tmp_path):
    from paper_2107_01391_b200 import _lib, build

    if not os.path.exists(_lib.LIB_PATH):
        build.build()
    exe = str(tmp_path / "test_facade")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "test_facade.cpp"), "-L", LIBDIR, "-lrecsort_b200",
                    "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_facade_builds(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_facade_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "OK" in r.stdout
