"""GPU: the C++ mirror of the reference API (include/bspsort_b200/bspsort.hpp)
compiled with the host compiler and run against libbsg.so."""
import os
import subprocess
import tempfile

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_api_restated_reference_tests(cuda):
    libdir = os.path.join(ROOT, "paper_1708_09495_b200")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "test_cpp_api")
        r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                            os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"), "-L", libdir, "-lbsg",
                            f"-Wl,-rpath,{libdir}", "-o", exe], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        assert r.stdout.startswith("OK"), r.stdout
