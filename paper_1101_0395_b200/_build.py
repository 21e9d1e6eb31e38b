"""In-tree build of libcqg.so (sm_100a only) with nvcc.

    python -m paper_1101_0395_b200._build        # or __graft_entry__.build()

Objects go to paper_1101_0395_b200/build/, the shared library to
paper_1101_0395_b200/libcqg.so (git-ignored; shipped to the GPU box by gpurun).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libcqg.so")
SOURCES = ["hist.cu", "lloyd.cu", "mapk.cu", "init.cu", "exact.cu", "api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def flags(extra=()) -> list[str]:
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                   "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, *extra]


def _newer(src_list, target) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def build(force: bool = False, verbose: bool = False, ptxas_info: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "cqg.h"))
    nv = nvcc()
    jobs = []
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _newer([s, *headers], o):
            extra = ["-Xptxas", "-v"] if ptxas_info else []
            jobs.append([nv, *flags(extra), "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for cmd, r in ex.map(run, jobs):
            if r.returncode != 0:
                raise RuntimeError("nvcc failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
            if verbose or ptxas_info:
                sys.stdout.write(r.stdout + r.stderr)
    if force or jobs or _newer(objs, LIB):
        cmd = [nv, *ARCH, "-shared", "--cudart", "static", "-o", LIB, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    build_host(force)
    return LIB


HOST_LIB = os.path.join(PKG, "libquant_b200.so")
CPP_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
CPP_TEST_BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")
CPP_E2E_SRC = os.path.join(ROOT, "tools", "cpp_e2e.cpp")
CPP_E2E_BIN = os.path.join(ROOT, "tools", "cpp_e2e")


HOST_SOURCES = ["context.cpp", "colour_rng.cpp", "image_io.cpp", "histogram_api.cpp", "cluster.cpp", "seeding.cpp",
                "report.cpp", "sweep.cpp"]


def build_host(force: bool = False) -> str:
    """libquant_b200.so: the reference's quant:: C++ API (include/quant/*.hpp)
    over libcqg.so, plus the C++ drop-in test binary."""
    cxx = shutil.which("g++") or "g++"
    inc = ["-I" + os.path.join(ROOT, "include")]
    host = os.path.join(PKG, "host")
    srcs = [os.path.join(host, f) for f in HOST_SOURCES]
    qdir = os.path.join(ROOT, "include", "quant")
    hdrs = [os.path.join(qdir, h) for h in os.listdir(qdir)] + [os.path.join(ROOT, "include", "cqg.h"),
                                                                 os.path.join(host, "context.hpp")]
    if force or _newer([*srcs, LIB, *hdrs], HOST_LIB):
        # -ffp-contract=off: no FMA contraction, like the reference's Release build
        cmd = [cxx, "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-shared", *inc, *srcs, "-o", HOST_LIB,
               "-L" + PKG, "-l:libcqg.so", "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("host library build failed:\n" + r.stdout + r.stderr)
    if force or _newer([CPP_TEST_SRC, HOST_LIB, *hdrs], CPP_TEST_BIN):
        cmd = [cxx, "-std=c++20", "-O2", *inc, CPP_TEST_SRC, "-o", CPP_TEST_BIN, "-L" + PKG, "-l:libquant_b200.so",
               "-l:libcqg.so", "-Wl,-rpath," + PKG]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("C++ test build failed:\n" + r.stdout + r.stderr)
    if force or _newer([CPP_E2E_SRC, HOST_LIB, *hdrs], CPP_E2E_BIN):
        cmd = [cxx, "-std=c++20", "-O2", *inc, CPP_E2E_SRC, "-o", CPP_E2E_BIN, "-L" + PKG, "-l:libquant_b200.so",
               "-l:libcqg.so", "-Wl,-rpath," + PKG]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("C++ e2e tool build failed:\n" + r.stdout + r.stderr)
    return HOST_LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, ptxas_info="--ptxas" in sys.argv))
