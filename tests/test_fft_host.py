"""CPU checks of the engine's FFT decomposition and shared-memory layout.

tests/host_fft_emu.cpp compiles the kernel's own per-thread pass functions
(paper_1910_01972_b200/csrc/olsb_fft.cuh) for the host and runs one segment
thread by thread.  This validates the window decomposition, the twiddle
forms (STD / GOOD / ROT, static junction constants) and the in-place index
maps against numpy and the oracle without a GPU.
"""

import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from conftest import ROOT, rel_err

CSRC = os.path.join(ROOT, "paper_1910_01972_b200", "csrc")


@pytest.fixture(scope="module")
def emu(tmp_path_factory):
    out = tmp_path_factory.mktemp("emu") / "libemu.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I", CSRC,
                    os.path.join(ROOT, "tests", "host_fft_emu.cpp"), "-o",
                    str(out)], check=True)
    lib = ctypes.CDLL(str(out))
    for fn in (lib.emu_fft_f, lib.emu_fft_d):
        fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                       ctypes.c_int]
    return lib


def _run(emu, x, inverse):
    n = x.shape[0]
    logn = n.bit_length() - 1
    out = np.empty_like(x)
    fn = emu.emu_fft_f if x.dtype == np.complex64 else emu.emu_fft_d
    assert fn(logn, x.ctypes.data, out.ctypes.data, int(inverse)) == 0
    return out


@pytest.mark.parametrize("logn", range(2, 13))
@pytest.mark.parametrize("dtype,tol", [(np.complex64, 2e-6),
                                       (np.complex128, 1e-14)])
def test_forward_matches_reference_layout(emu, logn, dtype, tol):
    n = 1 << logn
    rng = np.random.default_rng([1, logn])
    x = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(dtype)
    got = _run(emu, x, False)
    # same in-place positions as the reference's dif_fwd (bit-reversed)
    ref = oracle.fft_forward_permuted(x.astype(np.complex128), "double")
    assert rel_err(got, ref) < tol
    back = _run(emu, got, True)
    assert rel_err(back, x) < tol


@pytest.mark.parametrize("logn", [2, 5, 8, 11, 12])
def test_reorder_free_circular_convolution(emu, logn):
    # test_acceptance.py:146-160: inverse(fwd(a) * fwd(b)) = a (*) b
    n = 1 << logn
    rng = np.random.default_rng([2, logn])
    a = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    ref = np.fft.ifft(np.fft.fft(a) * np.fft.fft(b))
    fa = _run(emu, a.astype(np.complex64), False)
    fb = _run(emu, b.astype(np.complex64), False)
    got = _run(emu, (fa * fb).astype(np.complex64), True)
    assert rel_err(got, ref) < 1e-5


@pytest.mark.parametrize("dbl", [0, 1])
@pytest.mark.parametrize("logn", range(2, 13))
def test_smem_layout_conflict_free_and_injective(emu, dbl, logn):
    """Every exchange access of the kernel is bank-conflict free and the
    padded map is injective (kernel CTA = 256 threads = 256/T segments)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import smem_layout_search as S
    pd = (ctypes.c_int * 7)()
    emu.emu_pad(dbl, logn, pd)
    *kp, stride = list(pd)
    n = 1 << logn
    pos = [S.pos(p, *kp) for p in range(n)]
    assert len(set(pos)) == n and max(pos) < stride
    loge, logt, _, _, _ = S.geo(logn)
    segs = max(1, 256 >> logt)
    assert S.conflict_free(logn, min(segs, 64), *kp, stride, bool(dbl))


@pytest.mark.parametrize("dbl", [0, 1])
@pytest.mark.parametrize("logn", range(5, 13))
def test_exchange_layouts_conflict_free(emu, dbl, logn):
    """Every per-exchange layout (xpad_for) is injective, fits the buffer
    stride, keeps 128-bit pairs adjacent and 16-byte aligned, and is
    bank-conflict free for both window sides of the exchange."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import smem_layout_search as S
    loge, logt, npass, g0, los = S.geo(logn)
    if logt < 5:
        pytest.skip("several segments per warp: covered by the pad_for test")
    n = 1 << logn
    for x in range(npass - 1):
        v = (ctypes.c_int * 10)()
        emu.emu_xpad(dbl, logn, x, v)
        rb, k1, p1, k2, p2, k3, p3, plo, phi, span = list(v)
        kp = [k1, p1, k2, p2, k3, p3]
        pos = [S.xpos(p, rb, kp) for p in range(n)]
        assert len(set(pos)) == n and max(pos) < span
        if dbl:
            continue   # fp64 keeps pad_for (checked above)
        sides = [(x, None if plo < 0 else plo), (x + 1, None if phi < 0 else phi)]
        assert S.xconflict_free(logn, rb, kp, sides)
