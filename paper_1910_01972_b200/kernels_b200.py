"""The reference's kernel plugin seam, backed by the B200 engine.

olsconv picks its kernel module ``K`` at import (``backend.py:18-36``); both
of its backends export the same functions with numpy arguments
(``backend.py:11-12``).  This module is that third backend: same names, same
argument lists and meanings, same in-place / write-only-your-windows
contract, but every call runs on the GPU through the C ABI of
``include/olsb.h``.  A maintainer wires it in with one branch in
``backend.py``:

    elif _flag == "b200":
        from paper_1910_01972_b200 import kernels_b200 as kernels

Contract kept from ``_kernels_nb.py``:

* ``dif_fwd_batch(mat, tw)`` / ``dit_inv_batch(mat, twc)`` transform every
  row of ``mat`` IN PLACE (``_kernels_nb.py:54-63``);
* ``fused_c2c`` / ``fused_c2c_abs2`` / ``fused_r2r`` write ONLY the output
  windows of segments ``[seg_lo, seg_hi)`` of ``out`` (``:265-337``): the
  reference runs them concurrently on disjoint segment ranges
  (``ols.py:212-225``), so no other element of ``out`` may change;
* kernels never raise for valid arguments (the reference validates in
  Python first); a CUDA or engine error surfaces as ``EngineError``.

``EXACT`` (default on) selects the engine's exact mode where it exists:
``dif_fwd_batch``, ``fused_c2c`` (postproc none / scale) and
``fused_c2c_abs2`` then use the reference's own twiddle table and
operation order and are bit-identical to the numba kernels.  The other
calls (and ``EXACT = False``) run the fast engine, which agrees with the
reference within the stated fp32 tolerance.

Data moves per call (host numpy in, host numpy out) to honour the numpy
contract; code that keeps data on the GPU uses the package API instead
(``paper_1910_01972_b200.convolve``), which is what ``bench.py`` measures.
The scratch arguments (``buf``, ``spec_buf``, ``rbuf``, ...) are accepted
and unused: the engine keeps its scratch in registers, shared and tensor
memory.
"""

from __future__ import annotations

import threading
from typing import Dict, Tuple

import numpy as np
import torch

from . import _lib
from .errors import EngineError

EXACT = True

PP_NONE, PP_SCALE, PP_MAG2, PP_DERIV = 0, 1, 2, 3

_LOCK = threading.Lock()
# device copies of read-only (cached FilterSet) spectra, keyed by buffer
_SPEC_CACHE: Dict[Tuple, torch.Tensor] = {}


def _prec(a: np.ndarray) -> int:
    return 0 if a.dtype in (np.complex64, np.float32) else 1


def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise EngineError("the b200 kernel backend needs a CUDA device")
    return torch.device("cuda", torch.cuda.current_device())


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _to_dev(a: np.ndarray) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if not a.flags.writeable:       # torch wants writable host memory
        a = a.copy()
    return torch.from_numpy(a).to(_dev())


def _bitrev_perm(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    i = np.arange(n)
    r = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        r |= ((i >> b) & 1) << (bits - 1 - b)
    return r


def _engine_spectra(spectra: np.ndarray, n: int, key_extra=()) -> torch.Tensor:
    """Permuted complex spectra (rows of length n) -> engine layout on the
    device (olsb_spectra_perm_to_dev).  Read-only arrays (the reference's
    cached FilterSet spectra, ``ols.py:199-205``) are converted once."""
    key = None
    if not spectra.flags.writeable:
        key = (spectra.__array_interface__["data"][0], spectra.shape,
               spectra.dtype.str, n, torch.cuda.current_device()) + tuple(key_extra)
        with _LOCK:
            hit = _SPEC_CACHE.get(key)
        if hit is not None:
            return hit
    sp = _to_dev(spectra)
    dev = torch.empty((spectra.shape[0], _lib.load().olsb_spectra_dev_len(n)),
                      dtype=sp.dtype, device=sp.device)
    _lib.call("olsb_spectra_perm_to_dev", sp.data_ptr(), spectra.shape[0], n,
              dev.data_ptr(), _prec(spectra), _stream())
    if key is not None:
        with _LOCK:
            _SPEC_CACHE[key] = dev
    return dev


def _window_io(x: np.ndarray, out: np.ndarray, l_eff: int, seg_lo: int,
               seg_hi: int):
    """Device copies for one call: the whole signal, and a device tile for
    the output windows [g_lo, g_hi) of every filter."""
    n_s = x.shape[0]
    g_lo = seg_lo * l_eff
    g_hi = min(seg_hi * l_eff, n_s)
    xd = _to_dev(x)
    od = torch.empty((out.shape[0], max(1, g_hi - g_lo)),
                     dtype=torch.from_numpy(out[:1, :1]).dtype, device=xd.device)
    return xd, od, g_lo, g_hi


def _write_back(out: np.ndarray, od: torch.Tensor, g_lo: int, g_hi: int):
    if g_hi > g_lo:
        out[:, g_lo:g_hi] = od[:, :g_hi - g_lo].cpu().numpy()


# ---------------------------------------------------------------------------
# transforms (_kernels_nb.py:54-63)
# ---------------------------------------------------------------------------

def dif_fwd_batch(mat: np.ndarray, tw: np.ndarray) -> None:
    """Forward radix-2 DIF of every row, in place, bit-reversed output
    (``_kernels_nb.py:54-57``).  EXACT: the reference's table ``tw`` and
    operation order (bit-identical)."""
    rows, n = mat.shape
    if rows == 0:
        return
    d = _to_dev(mat)
    o = torch.empty_like(d)
    if EXACT:
        twd = _to_dev(np.asarray(tw, dtype=mat.dtype))
        _lib.call("olsb_filter_spectra_c2c_ref", d.data_ptr(), rows, n, n,
                  twd.data_ptr(), o.data_ptr(), None, _prec(mat), _stream())
    else:
        _lib.call("olsb_dif_fwd_batch", d.data_ptr(), o.data_ptr(), rows, n,
                  _prec(mat), _stream())
    mat[...] = o.cpu().numpy()


def dit_inv_batch(mat: np.ndarray, twc: np.ndarray) -> None:
    """Inverse radix-2 DIT of every row, in place, bit-reversed input,
    natural output, times 1/n (``_kernels_nb.py:60-63``); fast engine."""
    rows, n = mat.shape
    if rows == 0:
        return
    d = _to_dev(mat)
    o = torch.empty_like(d)
    _lib.call("olsb_dit_inv_batch", d.data_ptr(), o.data_ptr(), rows, n,
              _prec(mat), _stream())
    mat[...] = o.cpu().numpy()


# ---------------------------------------------------------------------------
# fused kernels (_kernels_nb.py:265-337)
# ---------------------------------------------------------------------------

def fused_c2c(x, spectra, tw, twc, m, origin, l_eff, t0, win_off,
              seg_lo, seg_hi, pp_kind, pp_c, h0, out, buf, spec_buf) -> None:
    """``K.fused_c2c`` (``_kernels_nb.py:265-285``): segments [seg_lo,
    seg_hi) of x, every filter; writes only those windows of ``out``."""
    n_s, n = x.shape[0], spectra.shape[1]
    if seg_hi <= seg_lo or spectra.shape[0] == 0:
        return
    sd = _engine_spectra(spectra, n)
    xd, od, g_lo, g_hi = _window_io(x, out, l_eff, seg_lo, seg_hi)
    if pp_kind == PP_DERIV and m == 1:
        # tap length 1 leaves no aliased sample for a halo in the reference's
        # geometry (it recomputes the seam neighbours from the input, _store
        # :232-260); the range entry's derivative geometry (t0 = 1, L = N -
        # 2) keeps both neighbours inside every segment
        _range_deriv("olsb_fused_c2c_range", xd, sd, spectra.shape[0], n, m,
                     origin, pp_c, od, g_lo, g_hi, x)
        _write_back(out, od, g_lo, g_hi)
        return
    common = (xd.data_ptr(), 0, n_s, sd.data_ptr(), spectra.shape[0], n, m,
              origin, l_eff, t0, win_off, seg_lo, seg_hi, int(pp_kind),
              float(pp_c))
    tail = (od.data_ptr(), od.shape[1], g_lo, _prec(x), _stream())
    if EXACT and pp_kind in (PP_NONE, PP_SCALE):
        twd = _to_dev(np.asarray(tw, dtype=x.dtype))
        _lib.call("olsb_fused_c2c_ref", *common, twd.data_ptr(), *tail)
    else:
        _lib.call("olsb_fused_c2c", *common, *tail)
    _write_back(out, od, g_lo, g_hi)


def fused_c2c_abs2(x, spectra, tw, twc, m, origin, l_eff, t0, win_off,
                   seg_lo, seg_hi, h0, out, buf, spec_buf) -> None:
    """``K.fused_c2c_abs2`` (``_kernels_nb.py:288-309``): |y|^2 into the
    real ``out``, windows of [seg_lo, seg_hi) only."""
    n_s, n = x.shape[0], spectra.shape[1]
    if seg_hi <= seg_lo or spectra.shape[0] == 0:
        return
    sd = _engine_spectra(spectra, n)
    xd, od, g_lo, g_hi = _window_io(x, out, l_eff, seg_lo, seg_hi)
    common = (xd.data_ptr(), 0, n_s, sd.data_ptr(), spectra.shape[0], n, m,
              origin, l_eff, t0, win_off, seg_lo, seg_hi)
    tail = (od.data_ptr(), od.shape[1], g_lo, _prec(x), _stream())
    if EXACT:
        twd = _to_dev(np.asarray(tw, dtype=x.dtype))
        _lib.call("olsb_fused_c2c_abs2_ref", *common, twd.data_ptr(), *tail)
    else:
        _lib.call("olsb_fused_c2c_abs2", *common, *tail)
    _write_back(out, od, g_lo, g_hi)


def fused_r2r(x, spectra, tw_half, tw_half_conj, pack_tw, pack_tw_conj,
              m, origin, l_eff, t0, win_off, seg_lo, seg_hi,
              pp_kind, pp_c, h0, out, rbuf, z_scr, bins, prod) -> None:
    """``K.fused_r2r`` (``_kernels_nb.py:312-337``): real signal, the real
    taps' ``rfft`` bins (n/2 + 1, natural order) as ``spectra``.  The engine
    multiplies by the full complex spectrum of the real taps: rebuilt here
    by Hermitian symmetry and bit-reversed into the permuted layout."""
    n_s = x.shape[0]
    h = spectra.shape[1] - 1
    n = 2 * h
    if seg_hi <= seg_lo or spectra.shape[0] == 0:
        return
    cdt = np.complex64 if x.dtype == np.float32 else np.complex128
    full = np.empty((spectra.shape[0], n), dtype=cdt)
    full[:, :h + 1] = spectra
    full[:, h + 1:] = np.conj(spectra[:, 1:h][:, ::-1])
    perm = full[:, _bitrev_perm(n)]
    if not spectra.flags.writeable:
        perm.flags.writeable = False
    sd = _engine_spectra(perm, n, key_extra=("r2r",
                                             spectra.__array_interface__["data"][0]))
    xd, od, g_lo, g_hi = _window_io(x, out, l_eff, seg_lo, seg_hi)
    if pp_kind == PP_DERIV and m == 1:     # as fused_c2c
        _range_deriv("olsb_fused_r2r_range", xd, sd, spectra.shape[0], n, m,
                     origin, pp_c, od, g_lo, g_hi, x)
        _write_back(out, od, g_lo, g_hi)
        return
    _lib.call("olsb_fused_r2r", xd.data_ptr(), 0, n_s, sd.data_ptr(),
              spectra.shape[0], n, m, origin, l_eff, t0, win_off, seg_lo,
              seg_hi, int(pp_kind), float(pp_c), od.data_ptr(), od.shape[1],
              g_lo, _prec(x), _stream())
    _write_back(out, od, g_lo, g_hi)


def _range_deriv(entry, xd, sd, n_fil, n, m, origin, pp_c, od, g_lo, g_hi, x):
    """Outputs [g_lo, g_hi) with the derivative epilogue through the range
    entry (olsb_fused_{c2c,r2r}_range, halo geometry) into the tile ``od``."""
    if g_hi <= g_lo:
        return
    _lib.call(entry, xd.data_ptr(), 0, x.shape[0], sd.data_ptr(), n_fil, n, m,
              origin, g_lo, g_hi, PP_DERIV, float(pp_c), od.data_ptr(),
              od.shape[1], g_lo, _prec(x), _stream())
