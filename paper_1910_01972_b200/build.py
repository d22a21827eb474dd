"""Build the in-tree CUDA library ``libolsb.so`` for sm_100a with nvcc.

    python -m paper_1910_01972_b200.build [--verbose]

The library is a plain C-ABI shared object (include/olsb.h) loaded with
ctypes; no torch headers are involved.  The kernel instantiations of each FFT
length are a separate object (olsb_inst.cu, -DOLSB_LOGN=L) compiled in
parallel, then linked with the C ABI (olsb_kernels.cu).  The .so travels to
the GPU box inside the repo snapshot.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libolsb.so")
SOURCES = [os.path.join(CSRC, "olsb_kernels.cu"),
           os.path.join(CSRC, "olsb_inst.cu")]
HEADERS = [os.path.join(CSRC, h) for h in
           ("olsb_fft.cuh", "olsb_engine.cuh", "olsb_w64.cuh", "olsb_w64x2.cuh", "olsb_w32x2.cuh", "olsb_launch.cuh")] + [
    os.path.join(INCLUDE, "olsb.h")]
LOGNS = range(2, 13)
OBJDIR = os.path.join(PKG, "build_obj")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the OLS engine has no non-CUDA path")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS)


def _run(cmd, verbose):
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libolsb.so")
    return res.stderr if verbose else ""


def build(verbose: bool = False, force: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    base = [nvcc(), *NVCC_FLAGS, "-I", INCLUDE, "-I", CSRC,
            *os.environ.get("OLSB_NVCC_EXTRA", "").split()]
    if verbose:
        base += ["-Xptxas", "-v"]
    jobs = [(base + ["-c", SOURCES[0], "-o",
                     os.path.join(OBJDIR, "olsb_kernels.o")])]
    for lg in LOGNS:
        jobs.append(base + [f"-DOLSB_LOGN={lg}", "-c", SOURCES[1], "-o",
                            os.path.join(OBJDIR, f"olsb_inst_{lg}.o")])
    # longest (largest N) first
    jobs = [jobs[0]] + jobs[1:][::-1]
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        logs = list(ex.map(lambda c: _run(c, verbose), jobs))
    objs = [j[-1] for j in jobs]
    _run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
          *objs, "-o", LIB + ".tmp", "-lcudart"], False)
    if verbose:
        sys.stderr.write("".join(logs))
    os.replace(LIB + ".tmp", LIB)
    return LIB


CUFFT_SRC = os.path.join(CSRC, "olsb_cufft.cu")
CUFFT_LIB = os.path.join(PKG, "libolsb_cufft.so")


def build_cufft(force: bool = False) -> str:
    """libolsb_cufft.so: the paper's cuFFT-OLS comparison point
    (csrc/olsb_cufft.cu), linked against the dynamic libcufft so the
    process's already-loaded cuFFT (torch's) is reused."""
    if (not force and os.path.exists(CUFFT_LIB)
            and os.path.getmtime(CUFFT_LIB) >= os.path.getmtime(CUFFT_SRC)):
        return CUFFT_LIB
    cudalib = os.path.join(os.path.dirname(os.path.dirname(nvcc())), "lib64")
    _run([nvcc(), *NVCC_FLAGS, "-I", INCLUDE, "-I", CSRC, "-shared", CUFFT_SRC,
          "-o", CUFFT_LIB + ".tmp", "-L", cudalib, "-lcufft",
          "-Xlinker", f"-rpath={cudalib}"], False)
    os.replace(CUFFT_LIB + ".tmp", CUFFT_LIB)
    return CUFFT_LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    args = ap.parse_args()
    print(build(verbose=args.verbose, force=args.force))
    print(build_cufft(force=args.force))
