"""CPU oracle for the fused OLS path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` arm may import this package, and only as the checker or
the timed CPU baseline: the product package never imports it (enforced by
tests/test_boundary.py).

It is a restatement of the reference (olsconv, /root/reference/pkg/src) in C
(oracle/ols_oracle.c, built by oracle/Makefile into oracle/build/) plus the
reference's integer planner restated in Python.  Pinning: the restatement is
checked against fixtures produced by the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz) in tests/test_oracle.py —
bit-exact in single precision for the transforms and the fused path.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libolsoracle.so")
_LIB = None
_LOCK = threading.Lock()

c_vp, c_int, c_i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64


def build() -> str:
    """Compile the C restatement (gcc only; no reference sources involved)."""
    src = os.path.join(HERE, "ols_oracle.c")
    if (not os.path.exists(LIB_PATH)
            or os.path.getmtime(src) > os.path.getmtime(LIB_PATH)):
        subprocess.run(["make", "-C", HERE, "-B"], check=True,
                       capture_output=True)
    return LIB_PATH


def lib():
    global _LIB
    with _LOCK:
        if _LIB is None:
            if not os.path.exists(LIB_PATH):
                build()
            L = ctypes.CDLL(LIB_PATH)
            for sfx, R in (("f", ctypes.c_float), ("d", ctypes.c_double)):
                getattr(L, f"ols_tables_{sfx}").argtypes = [c_int, c_vp, c_vp]
                getattr(L, f"ols_dif_fwd_batch_{sfx}").argtypes = [c_vp, c_int, c_int, c_vp]
                getattr(L, f"ols_dit_inv_batch_{sfx}").argtypes = [c_vp, c_int, c_int, c_vp]
                getattr(L, f"ols_fused_c2c_{sfx}").argtypes = [
                    c_vp, c_i64, c_vp, c_int, c_int, c_vp, c_vp, c_i64, c_i64,
                    c_i64, c_i64, c_i64, c_int, ctypes.c_double, c_vp, c_int]
            L.ols_direct_d.argtypes = [c_vp, c_i64, c_vp, c_int, c_int, c_int,
                                       c_vp, c_int]
            L.ols_oracle_max_threads.restype = c_int
            _LIB = L
        return _LIB


def max_threads() -> int:
    return lib().ols_oracle_max_threads()


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _cdtype(precision: str):
    return np.complex64 if precision == "single" else np.complex128


def _sfx(precision: str) -> str:
    return "f" if precision == "single" else "d"


def tables(n: int, precision: str = "single"):
    """tw, twc of make_plan(n, "ct_dif_permuted") (fft.py:70-99)."""
    tw = np.empty(n // 2, _cdtype(precision))
    twc = np.empty_like(tw)
    getattr(lib(), f"ols_tables_{_sfx(precision)}")(n, _ptr(tw), _ptr(twc))
    return tw, twc


def fft_forward_permuted(rows, precision: str = "single") -> np.ndarray:
    """K.dif_fwd (_kernels_nb.py:11-28) on each row; bit-reversed out."""
    a = np.array(rows, dtype=_cdtype(precision), ndmin=2, copy=True)
    tw, _ = tables(a.shape[1], precision)
    getattr(lib(), f"ols_dif_fwd_batch_{_sfx(precision)}")(
        _ptr(a), a.shape[0], a.shape[1], _ptr(tw))
    return a if np.ndim(rows) == 2 else a[0]


def fft_inverse_permuted(rows, precision: str = "single") -> np.ndarray:
    """K.dit_inv (_kernels_nb.py:31-51) on each row; natural out, x 1/n."""
    a = np.array(rows, dtype=_cdtype(precision), ndmin=2, copy=True)
    _, twc = tables(a.shape[1], precision)
    getattr(lib(), f"ols_dit_inv_batch_{_sfx(precision)}")(
        _ptr(a), a.shape[0], a.shape[1], _ptr(twc))
    return a if np.ndim(rows) == 2 else a[0]


def plan(ns: int, m: int, n: int):
    """(valid_len, n_segments) of ols.plan (ols.py:116-117)."""
    valid = n - m + 1
    return valid, -(-ns // valid)


def geometry(m: int, origin: int, n: int):
    """_geometry with no halo (ols.py:133-136): (l_eff, t0, win_off)."""
    return n - m + 1, m - 1, origin - (m - 1)


def transform_filters(taps, n: int, precision: str = "single") -> np.ndarray:
    """transform_filters(..., "permuted") c2c (ols.py:194-199)."""
    taps = np.asarray(taps)
    padded = np.zeros((taps.shape[0], n), _cdtype(precision))
    padded[:, :taps.shape[1]] = taps
    return fft_forward_permuted(padded, precision)


def fused_convolve(x, taps, n: int, origin: int = 0,
                   precision: str = "single", threads: int = 0,
                   seg_lo: int = 0, seg_hi=None, pp_kind: int = 0,
                   pp_c: float = 1.0, out=None) -> np.ndarray:
    """convolve(variant="fused") c2c (ols.py:257-360 -> fused_c2c).  With
    seg_lo/seg_hi only those segments' output windows are written (the rest
    of ``out`` is left as given; NaN when allocated here)."""
    dt = _cdtype(precision)
    x = np.ascontiguousarray(x, dtype=dt)
    taps = np.asarray(taps)
    n_fil, m = taps.shape
    ns = x.shape[0]
    l_eff, t0, win_off = geometry(m, origin, n)
    _, n_seg = plan(ns, m, n)
    seg_hi = n_seg if seg_hi is None else seg_hi
    spectra = transform_filters(taps, n, precision)
    tw, twc = tables(n, precision)
    if out is None:
        out = np.full((n_fil, ns), np.nan, dt)
    threads = threads or max_threads()
    getattr(lib(), f"ols_fused_c2c_{_sfx(precision)}")(
        _ptr(x), ns, _ptr(spectra), n_fil, n, _ptr(tw), _ptr(twc), l_eff, t0,
        win_off, seg_lo, seg_hi, pp_kind, pp_c, _ptr(out), threads)
    return out


def direct_convolve(x, taps, origin: int = 0, threads: int = 0) -> np.ndarray:
    """oracle_conv (_kernels_nb.py:183-199), complex128 accumulate."""
    x = np.ascontiguousarray(x, dtype=np.complex128)
    taps = np.ascontiguousarray(taps, dtype=np.complex128)
    n_fil, m = taps.shape
    out = np.empty((n_fil, x.shape[0]), np.complex128)
    lib().ols_direct_d(_ptr(x), x.shape[0], _ptr(taps), n_fil, m, origin,
                       _ptr(out), threads or max_threads())
    return out


def direct_window(x, taps, origin: int, a: int, b: int,
                  threads: int = 0) -> np.ndarray:
    """Ground truth of outputs [a, b) only: y[:, a:b] depends on
    x[a - (m-1) + origin, b + origin) (zero-extended), SURVEY §8(c)."""
    x = np.asarray(x)
    taps = np.asarray(taps)
    m = taps.shape[1]
    lo = a - (m - 1) + origin
    hi = b + origin
    sub = np.zeros(hi - lo, np.complex128)
    s0, s1 = max(lo, 0), min(hi, x.shape[0])
    if s1 > s0:
        sub[s0 - lo:s1 - lo] = x[s0:s1]
    y = direct_convolve(sub, taps, m - 1, threads)
    return y[:, :b - a]
