"""CPU tests of the boundary: the C-ABI library builds for sm_100a, loads
without a GPU, exports every symbol include/scmoe.h declares, and its SASS
has the properties the design relies on (no FMA in the exact-order GEMM,
tcgen05 MMA + TMA in the grouped GEMM)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "scmoe.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(scmoe_\w+)\s*\(", hdr)))


@pytest.fixture(scope="module")
def built():
    from paper_2509_01322_b200 import build as B
    return B.build()


def test_library_exports_every_declared_symbol(built):
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\sT\s(scmoe_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_python_binding_covers_header(built):
    import paper_2509_01322_b200 as P
    assert set(declared_symbols()) <= set(P.exported_symbols())
    L = P.lib()  # loads without a GPU
    assert L.scmoe_version().decode().startswith("scmoe-b200")


def test_no_device_means_loud_failure(built):
    import paper_2509_01322_b200 as P
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(P.DeviceError):
        P.Context(0)


def test_sass_properties(built):
    from paper_2509_01322_b200 import build as B
    summary = B.check_sass(built)
    seq = [k for k in summary if re.search(r"seq_gemm_kernel.*Lb0E", k)]
    assert seq and all(summary[k]["FFMA"] == 0 for k in seq)
    gemm = [k for k in summary if "grouped_gemm_kernel" in k]
    assert gemm and all(summary[k]["UTCHMMA"] > 0 and summary[k]["UTMALDG"] > 0 and
                        summary[k]["LDTM"] > 0 for k in gemm)


def test_compat_header_compiles(built):
    """The C++ drop-in tier (include/moelab_b200) compiles against the C ABI."""
    src = os.path.join(ROOT, "tests", "cpp", "compat_smoke.cpp")
    if not os.path.exists(src):
        pytest.skip("compat smoke not present")
    exe = os.path.join(ROOT, "paper_2509_01322_b200", "_build", "compat_smoke")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), src, "-o",
                    exe, "-L" + os.path.dirname(built), "-lscmoe",
                    "-Wl,-rpath," + os.path.dirname(built)], check=True)
