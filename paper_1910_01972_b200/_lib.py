"""ctypes binding of the C ABI in include/olsb.h (libolsb.so, built in-tree).

There is no fallback: if the library is missing or cannot be loaded, every
engine call raises.  ``load()`` builds the library first when nvcc is present
and the sources are newer (development convenience; the GPU box receives the
prebuilt .so with the repo snapshot).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import EngineError

_LOCK = threading.Lock()
_LIB = None
LIB_PATH = os.environ.get("OLSB_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libolsb.so")

c_int, c_i64, c_vp, c_dbl = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double

# name -> (restype, argtypes); every symbol declared in include/olsb.h
SIGNATURES = {
    "olsb_version": (c_int, []),
    "olsb_error_string": (ctypes.c_char_p, [c_int]),
    "olsb_spectra_dev_len": (c_int, [c_int]),
    "olsb_dif_fwd_batch": (c_int, [c_vp, c_vp, c_int, c_int, c_int, c_vp]),
    "olsb_dit_inv_batch": (c_int, [c_vp, c_vp, c_int, c_int, c_int, c_vp]),
    "olsb_filter_spectra_c2c": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_vp,
                                        c_int, c_vp]),
    "olsb_spectra_perm_to_dev": (c_int, [c_vp, c_int, c_int, c_vp, c_int, c_vp]),
    "olsb_fused_c2c": (c_int, [c_vp, c_i64, c_i64, c_vp, c_int, c_int, c_int,
                               c_int, c_i64, c_int, c_i64, c_i64, c_i64, c_int,
                               c_dbl, c_vp, c_i64, c_i64, c_int, c_vp]),
    "olsb_fused_c2c_range": (c_int, [c_vp, c_i64, c_i64, c_vp, c_int, c_int,
                                     c_int, c_int, c_i64, c_i64, c_int, c_dbl,
                                     c_vp, c_i64, c_i64, c_int, c_vp]),
    "olsb_fused_c2c_ref": (c_int, [c_vp, c_i64, c_i64, c_vp, c_int, c_int,
                                   c_int, c_int, c_i64, c_int, c_i64, c_i64,
                                   c_i64, c_int, c_dbl, c_vp, c_vp, c_i64,
                                   c_i64, c_int, c_vp]),
    "olsb_fused_c2c_abs2_ref": (c_int, [c_vp, c_i64, c_i64, c_vp, c_int,
                                        c_int, c_int, c_int, c_i64, c_int,
                                        c_i64, c_i64, c_i64, c_vp, c_vp,
                                        c_i64, c_i64, c_int, c_vp]),
    "olsb_filter_spectra_c2c_ref": (c_int, [c_vp, c_int, c_int, c_int, c_vp,
                                            c_vp, c_vp, c_int, c_vp]),
    "olsb_fused_c2c_abs2": (c_int, [c_vp, c_i64, c_i64, c_vp, c_int, c_int,
                                    c_int, c_int, c_i64, c_int, c_i64, c_i64,
                                    c_i64, c_vp, c_i64, c_i64, c_int, c_vp]),
    "olsb_fused_r2r": (c_int, [c_vp, c_i64, c_i64, c_vp, c_int, c_int, c_int,
                               c_int, c_i64, c_int, c_i64, c_i64, c_i64, c_int,
                               c_dbl, c_vp, c_i64, c_i64, c_int, c_vp]),
    "olsb_fused_r2r_range": (c_int, [c_vp, c_i64, c_i64, c_vp, c_int, c_int,
                                     c_int, c_int, c_i64, c_i64, c_int, c_dbl,
                                     c_vp, c_i64, c_i64, c_int, c_vp]),
    "olsb_input_extent": (c_int, [c_int, c_int, c_int, c_i64, c_i64,
                                  ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "olsb_input_extent_pp": (c_int, [c_int, c_int, c_int, c_int, c_int, c_i64,
                                     c_i64, ctypes.POINTER(c_i64),
                                     ctypes.POINTER(c_i64)]),
    "olsb_input_extent_r2r": (c_int, [c_int, c_int, c_int, c_i64, c_i64,
                                      ctypes.POINTER(c_i64),
                                      ctypes.POINTER(c_i64)]),
    "olsb_set_filter_chunk": (c_int, [c_int]),
    "olsb_copy2d_async": (c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64,
                                  c_int, c_vp]),
}


def load(build_if_stale: bool = True):
    """Load (and if needed build) libolsb.so; raise if unavailable."""
    global _LIB
    with _LOCK:
        if _LIB is not None:
            return _LIB
        if build_if_stale:
            try:
                from . import build as _build
                if _build.needs_build():
                    _build.build()
            except RuntimeError:
                if not os.path.exists(LIB_PATH):
                    raise
        if not os.path.exists(LIB_PATH):
            raise EngineError(
                f"{LIB_PATH} is missing; run `python -m "
                "paper_1910_01972_b200.build` (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        lib = load()
        msg = lib.olsb_error_string(rc).decode()
        raise EngineError(f"{what} failed: {msg} (code {rc})")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
