"""ctypes binding of libolsb_cufft.so: the cuFFT-based OLS comparison
point (csrc/olsb_cufft.cu).  Like libolsb.so it has no fallback: a missing
library raises."""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from .errors import EngineError

_LOCK = threading.Lock()
_LIB = None
_WORK = {}
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                        "libolsb_cufft.so")


def load():
    global _LIB
    with _LOCK:
        if _LIB is None:
            if not os.path.exists(LIB_PATH):
                from .build import build_cufft
                build_cufft()
            L = ctypes.CDLL(LIB_PATH)
            vp, i, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
            L.olsb_cufft_ols_workspace.restype = ctypes.c_size_t
            L.olsb_cufft_ols_workspace.argtypes = [i64, i, i, i]
            L.olsb_cufft_ols_c2c.restype = i
            L.olsb_cufft_ols_c2c.argtypes = [vp, i64, vp, i, i, i, i, vp, i64,
                                             vp, vp]
            _LIB = L
        return _LIB


def ols_c2c(x, n_s, spectra, n_fil, n, m, origin, out, out_ld, stream):
    L = load()
    need = L.olsb_cufft_ols_workspace(n_s, n_fil, n, m)
    work = _WORK.get(x.device.index)
    if work is None or work.numel() < need:
        work = torch.empty(need, dtype=torch.uint8, device=x.device)
        _WORK[x.device.index] = work
    rc = L.olsb_cufft_ols_c2c(x.data_ptr(), n_s, spectra.data_ptr(), n_fil, n,
                              m, origin, out.data_ptr(), out_ld,
                              work.data_ptr(), stream)
    if rc != 0:
        raise EngineError(f"olsb_cufft_ols_c2c failed ({rc})")
