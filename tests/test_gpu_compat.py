"""The C++ drop-in tier on the GPU: the reference's own hot-path unit tests,
restated in tests/cpp/compat_smoke.cpp against include/moelab_b200/moelab.hpp,
compiled and run through libscmoe.so."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_compat_reference_unit_cases(scmoe):
    lib = os.path.join(ROOT, "paper_2509_01322_b200")
    exe = os.path.join(lib, "_build", "compat_smoke")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "compat_smoke.cpp"), "-o", exe, "-L" + lib,
                    "-lscmoe", "-Wl,-rpath," + lib], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
