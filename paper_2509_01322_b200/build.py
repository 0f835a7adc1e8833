"""Build libscmoe.so (sm_100a) in-tree.

    python -m paper_2509_01322_b200.build [--force]

Every .cu is compiled with ``-gencode arch=compute_100a,code=sm_100a``
(plain ``-arch=sm_100a`` also emits compute_100 PTX, which rejects tcgen05;
SURVEY.md 0.8a).  The exact-order kernels are additionally compiled with
``--fmad=false`` and the build asserts from the SASS that the sequential-k
GEMM (router projection / fp32 expert path) contains no fused multiply-add
(SURVEY.md 0.8b-c), and that the grouped GEMM really issues tcgen05 MMAs
(UTCHMMA) fed by TMA (UTMALDG).
"""
from __future__ import annotations

import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libscmoe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUOBJDUMP = os.path.join(os.path.dirname(NVCC), "cuobjdump")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                 "-I" + os.path.join(ROOT, "include")]
SOURCES = {
    "kernels_router.cu": ["--fmad=false"],
    "router_sm100.cu": ["--fmad=false", "-Xptxas", "-O1"],
    "kernels_moe.cu": ["--fmad=false"],
    "mla.cu": ["--fmad=false"],
    "capi.cu": [],
    "gemm_sm100.cu": ["-Xptxas", "-v"],
    "ep.cu": [],
    "mla_tc.cu": [],
}
HOST_SOURCES = ["host_rng.cpp"]
HEADERS = ["internal.cuh", "libm_port.h", "sm100_util.cuh", "f32x2.cuh"]


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def check_sass(lib: str = LIB) -> dict:
    """Assert the SASS properties the design relies on; returns a summary."""
    sass = _run([CUOBJDUMP, "-sass", lib])
    funcs = re.split(r"\n\s+Function : ", sass)
    summary = {}
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        body = f
        summary[name] = {
            "FFMA": len(re.findall(r"\bFFMA2?\b", body)),
            "DFMA": len(re.findall(r"\bDFMA\b", body)),
            "UTCHMMA": len(re.findall(r"UTC\w*MMA", body)),
            "UTMALDG": len(re.findall(r"UTMALDG", body)),
            "LDTM": len(re.findall(r"\bLDTM", body)),
        }
    # The plain sequential-k GEMM (router projection, fp32 W_out GEMM) must be
    # pure FMUL + FADD.  The SiLU instantiation's only FFMAs come from the
    # correctly rounded IEEE division (__fdiv_rn) inside the logistic.
    seq = [n for n in summary if re.search(r"seq_gemm_kernel.*Lb0E", n)]
    seq += [n for n in summary if re.search(r"router_(tma|slab|lean)_kernel", n)]
    # MLA: the scores / rope kernels are pure FMUL + FADD; the PV kernel's only
    # FFMAs are the correctly rounded divisions w = e / denom (__fdiv_rn) where
    # it stages the weights -- its chains are FMUL2 + FADD2 (no FFMA2 below)
    seq += [n for n in summary if re.search(r"mla_(scores|scores_big|scale_rope)_kernel|seq_gemv_kernel", n)]
    assert seq, "seq_gemm kernel missing from SASS"
    for n in seq:
        assert summary[n]["FFMA"] == 0, f"{n}: FFMA found in exact-order kernel"
    # packed f32x2 is only ever used as separately rounded FMUL2 + FADD2 (the
    # half-swap trick, f32x2.cuh); a fused FFMA2 anywhere would be a contraction
    assert not re.search(r"\bFFMA2\b", sass), "FFMA2 found: an f32x2 mul+add was contracted"
    # the double-precision router projection: separately rounded DMUL + DADD
    for n in summary:
        if "router_f64_kernel" in n:
            assert summary[n]["DFMA"] == 0, f"{n}: DFMA found in exact-order kernel"
    gemm = [n for n in summary if "grouped_gemm_kernel" in n]
    assert gemm and all(summary[n]["UTCHMMA"] > 0 and summary[n]["UTMALDG"] > 0 for n in gemm), \
        "grouped GEMM lacks UTCHMMA/UTMALDG"
    return summary


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "scmoe.h")]
    jobs = []
    objs = []
    for src, extra in SOURCES.items():
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _newer([s] + headers, o):
            jobs.append([NVCC] + COMMON + extra + ["-c", s, "-o", o])
    for src in HOST_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _newer([s, os.path.join(ROOT, "include", "scmoe.h")], o):
            jobs.append(["g++", "-O3", "-std=c++17", "-fPIC", "-ffp-contract=off",
                         "-I" + os.path.join(ROOT, "include"), "-c", s, "-o", o])
    logs = []
    if jobs:
        with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            logs = list(ex.map(_run, jobs))
    if force or jobs or not os.path.exists(LIB) or _newer(objs, LIB):
        tmp = LIB + ".tmp"
        _run([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lpthread", "-ldl"])
        summary = check_sass(tmp)  # a library failing the SASS checks is never installed
        os.replace(tmp, LIB)
        with open(os.path.join(BUILD, "sass_summary.txt"), "w") as f:
            for k, v in sorted(summary.items()):
                f.write(f"{k}: {v}\n")
            f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
