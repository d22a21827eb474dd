"""Overlap-save planner and convolution engines (reference: olsconv/ols.py).

The planner and geometry are the reference's integer math, line for line in
behaviour (ols.py:53-155), so plans and output windows are identical.  The
engines run on the GPU:

* ``fused`` — the product: one sm_100a kernel per call (C ABI
  ``olsb_fused_c2c``) doing the paper's Algorithm 2 per segment: gather the
  overlapped window, forward FFT in registers/shared memory, then per filter
  multiply with the cached spectrum, inverse FFT and write the valid samples.
* ``pipelined`` — the paper's cuFFT-OLS comparison point (Algorithm 1,
  reference _pipelined ols.py:363-410): gather segments, batched cuFFT C2C,
  a materialized (n_fil, rows, n) product, batched inverse cuFFT, discard.
  Chunked over segments so the product tensor fits a memory budget.
* ``full_fft_baseline`` — one padded cuFFT convolution of the whole signal.
* ``direct_oracle`` — direct time-domain convolution on the GPU in float64
  (the reference's ground-truth variant, oracle.py:20-41).

Segments write disjoint output windows, so any split of the segment range
(``workers`` launches, shards on several GPUs, host-streaming chunks) gives
bit-identical results.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable, List, Optional, Tuple

import numpy as np
import torch

from . import _lib
from .core import FilterSet, Precision, Signal, make_filterset, make_signal
from .errors import (BadLength, DomainMismatch, EngineError, FilterTooLong,
                     HaloUnavailable, LayoutMismatch, PlanMismatch,
                     SegmentTooSmall, TooLarge)
from .fft import DEFAULT_MAX_FFT_LEN
from .postproc import NONE, PostProcSpec

MODES = ("c2c", "r2r")
ENGINE_VARIANTS = ("fused", "pipelined", "full_fft_baseline", "direct_oracle",
                   "fused_exact", "cufft_ols")

DEFAULT_MAX_FULL_LEN = 1 << 25
PIPELINED_DEFAULT_SEGMENT = 8192
# bytes of the materialized cuFFT-OLS product tensor per chunk
PIPELINED_BUDGET_BYTES = 2 << 30


@dataclass(frozen=True)
class SegmentPlan:
    """Blocking geometry (ols.py:53-66): segment s reads the zero-extended
    input window [s*valid_len - (tap_len-1) + origin, ... + fft_len) and writes
    output window [s*valid_len, min((s+1)*valid_len, signal_len))."""

    fft_len: int
    tap_len: int
    valid_len: int
    n_segments: int
    signal_len: int
    mode: str
    origin: int


def next_pow2(n: int) -> int:
    return 1 if n <= 1 else 1 << (n - 1).bit_length()


def _is_pow2(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def auto_segment_len(tap_len: int, variant: str = "fused",
                     max_fft_len: int = DEFAULT_MAX_FFT_LEN) -> int:
    """Untuned default segment length (ols.py:76-87)."""
    if variant == "pipelined":
        return max(PIPELINED_DEFAULT_SEGMENT, next_pow2(tap_len))
    n = max(64, next_pow2(4 * (tap_len - 1)))
    return min(n, max_fft_len)


def plan(signal_len: int, tap_len: int, mode: str, origin: int = 0,
         fft_len: Optional[int] = None,
         max_fft_len: int = DEFAULT_MAX_FFT_LEN) -> SegmentPlan:
    """Overlap-save geometry with the reference's validation order and
    exceptions (ols.py:90-120)."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    if signal_len < 1 or tap_len < 1:
        raise ValueError("signal and filter must be non-empty")
    if not 0 <= origin <= tap_len - 1:
        raise ValueError(f"origin {origin} outside [0, {tap_len - 1}]")
    if tap_len > max_fft_len:
        raise FilterTooLong(
            f"tap length {tap_len} exceeds max segment length {max_fft_len};"
            " use full_fft_convolve")
    if fft_len is None or fft_len == "auto":
        n = auto_segment_len(tap_len, max_fft_len=max_fft_len)
    else:
        n = int(fft_len)
        floor = 8 if mode == "r2r" else 4
        if not _is_pow2(n) or n < floor:
            raise BadLength(
                f"segment length must be a power of two >= {floor}, got {n}")
        if n < tap_len:
            raise SegmentTooSmall(
                f"segment length {n} shorter than filter ({tap_len} taps)")
    valid = n - tap_len + 1
    n_seg = -(-signal_len // valid)
    return SegmentPlan(fft_len=n, tap_len=tap_len, valid_len=valid,
                       n_segments=n_seg, signal_len=signal_len, mode=mode,
                       origin=origin)


def _geometry(seg_plan: SegmentPlan, halo: int) -> Tuple[int, int, int, int]:
    """(l_eff, t0, win_off, n_seg_eff) for a post-processing halo
    (ols.py:123-146)."""
    m = seg_plan.tap_len
    o = seg_plan.origin
    if halo == 0 or m == 1:
        l_eff = seg_plan.valid_len
        t0 = m - 1
        win_off = o - (m - 1)
    else:
        l_eff = seg_plan.valid_len - 2 * halo
        t0 = m - 1 + halo
        win_off = o - (m - 1) - halo
        if l_eff < 1:
            raise HaloUnavailable(
                f"segment length {seg_plan.fft_len} leaves no room for a"
                f" halo of {halo} around {seg_plan.tap_len} taps")
    n_seg_eff = -(-seg_plan.signal_len // l_eff)
    return l_eff, t0, win_off, n_seg_eff


def output_windows(seg_plan: SegmentPlan,
                   postproc: PostProcSpec = NONE) -> List[Tuple[int, int]]:
    """Per-segment output windows: disjoint, covering [0, signal_len)
    (ols.py:149-155)."""
    l_eff, _, _, n_seg = _geometry(seg_plan, postproc.halo)
    n_s = seg_plan.signal_len
    return [(s * l_eff, min((s + 1) * l_eff, n_s)) for s in range(n_seg)]


def _chunk_bounds(n_items: int, workers: int) -> List[Tuple[int, int]]:
    """Contiguous item ranges (ols.py:212-215); also the multi-GPU shard map."""
    k = max(1, min(workers, n_items))
    step = -(-n_items // k)
    return [(lo, min(lo + step, n_items)) for lo in range(0, n_items, step)]


def _required_layout(mode: str, variant: str) -> str:
    return ("permuted" if (mode == "c2c" and variant in ("fused", "fused_exact"))
            else "natural")


def _stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


# ---------------------------------------------------------------------------
# filter spectra
# ---------------------------------------------------------------------------

def transform_filters(filters: FilterSet, seg_plan: SegmentPlan,
                      layout: str = "natural") -> FilterSet:
    """Zero-pad every filter to the segment length and cache its forward
    transform (ols.py:168-205).  "permuted" spectra come from the engine's own
    in-register FFT (olsb_filter_spectra_c2c), which also writes the coalesced
    engine layout the fused kernel streams."""
    if layout not in ("natural", "permuted"):
        raise ValueError(f"layout must be natural|permuted, got {layout!r}")
    if filters.tap_length != seg_plan.tap_len:
        raise PlanMismatch(
            f"filter tap length {filters.tap_length} != plan "
            f"{seg_plan.tap_len}")
    precision = (Precision.single
                 if filters.taps.dtype in (torch.float32, torch.complex64)
                 else Precision.double)
    n = seg_plan.fft_len
    taps = filters.taps
    if seg_plan.mode == "r2r":
        if filters.value_kind != "real":
            raise PlanMismatch("complex filter taps on the real path")
        if layout != "natural":
            raise LayoutMismatch("packed real spectra are natural-order only")
        # the engine's own in-register FFT of the real taps (zero imaginary
        # parts): the full complex spectrum, permuted + engine layout.  The
        # fused real engine multiplies by it (it transforms two real
        # segments as one complex segment); the host-visible spectra keep
        # the reference's packed rfft semantics (n/2 + 1 bins, natural
        # order, ols.py:183-193), read out of the permuted spectrum (bin k
        # sits at bit-reversed position rev(k))
        if n > 4096:
            # segment lengths beyond the engine's (the cuFFT comparison path
            # only): cuFFT's rfft
            padded = torch.zeros((filters.n_filters, n),
                                 dtype=precision.torch_real, device=taps.device)
            padded[:, :filters.tap_length] = taps
            return filters.with_spectra(torch.fft.rfft(padded, dim=1), layout, n)
        ctaps = taps.to(precision.torch_complex).contiguous()
        perm = torch.empty((filters.n_filters, n), dtype=precision.torch_complex,
                           device=taps.device)
        dev = torch.empty_like(perm)
        with torch.cuda.device(taps.device):
            _lib.call("olsb_filter_spectra_c2c", ctaps.data_ptr(),
                      filters.n_filters, filters.tap_length, n,
                      perm.data_ptr(), dev.data_ptr(), precision.code,
                      _stream_ptr())
        bins = perm[:, _bitrev_index(n, taps.device)[:n // 2 + 1]].contiguous()
        return filters.with_spectra(bins, layout, n, dev)
    ctaps = taps.to(precision.torch_complex).contiguous()
    if layout == "permuted":
        spectra = torch.empty((filters.n_filters, n),
                              dtype=precision.torch_complex, device=taps.device)
        dev = torch.empty_like(spectra)
        with torch.cuda.device(taps.device):
            _lib.call("olsb_filter_spectra_c2c", ctaps.data_ptr(),
                      filters.n_filters, filters.tap_length, n,
                      spectra.data_ptr(), dev.data_ptr(), precision.code,
                      _stream_ptr())
        return filters.with_spectra(spectra, layout, n, dev)
    if n <= 4096:
        # natural order (the comparison variants' layout): the engine's own
        # in-register FFT, read out of the permuted spectrum (bin k at
        # bit-reversed position rev(k)), as for the real path
        perm = torch.empty((filters.n_filters, n), dtype=precision.torch_complex,
                           device=taps.device)
        dev = torch.empty_like(perm)
        with torch.cuda.device(taps.device):
            _lib.call("olsb_filter_spectra_c2c", ctaps.data_ptr(),
                      filters.n_filters, filters.tap_length, n,
                      perm.data_ptr(), dev.data_ptr(), precision.code,
                      _stream_ptr())
        nat = perm[:, _bitrev_index(n, taps.device)].contiguous()
        return filters.with_spectra(nat, layout, n)
    # segment lengths beyond the engine's (comparison paths only): cuFFT
    padded = torch.zeros((filters.n_filters, n), dtype=precision.torch_complex,
                         device=taps.device)
    padded[:, :filters.tap_length] = ctaps
    return filters.with_spectra(torch.fft.fft(padded, dim=1), layout, n)


_BITREV = {}


def _bitrev_index(n: int, device) -> torch.Tensor:
    """rev(k) for k < n (log2 n bits): natural bin k of a permuted spectrum."""
    key = (n, str(device))
    t = _BITREV.get(key)
    if t is None:
        bits = n.bit_length() - 1
        k = torch.arange(n)
        r = torch.zeros(n, dtype=torch.int64)
        for b in range(bits):
            r |= ((k >> b) & 1) << (bits - 1 - b)
        t = r.to(device)
        _BITREV[key] = t
    return t


def _engine_spectra(filters: FilterSet) -> torch.Tensor:
    """Engine-layout spectra; converted once from a permuted cache that was
    filled elsewhere (e.g. handed over from the reference)."""
    if filters.spectra_dev is not None:
        return filters.spectra_dev
    if filters.spectra.shape[1] != filters.spectra_n:
        # packed real (rfft) spectra: the engine needs the full complex
        # spectrum of the real taps, recomputed by the engine's own FFT
        n = filters.spectra_n
        prec = (Precision.single if filters.taps.dtype == torch.float32
                else Precision.double)
        ctaps = filters.taps.to(prec.torch_complex).contiguous()
        dev = torch.empty((filters.n_filters, n), dtype=prec.torch_complex,
                          device=ctaps.device)
        with torch.cuda.device(ctaps.device):
            _lib.call("olsb_filter_spectra_c2c", ctaps.data_ptr(),
                      filters.n_filters, filters.tap_length, n, None,
                      dev.data_ptr(), prec.code, _stream_ptr())
        object.__setattr__(filters, "spectra_dev", dev)
        return dev
    spec = filters.spectra.contiguous()
    dev = torch.empty_like(spec)
    prec = Precision.single if spec.dtype == torch.complex64 else Precision.double
    _lib.call("olsb_spectra_perm_to_dev", spec.data_ptr(), spec.shape[0],
              spec.shape[1], dev.data_ptr(), prec.code, _stream_ptr())
    object.__setattr__(filters, "spectra_dev", dev)
    return dev


# ---------------------------------------------------------------------------
# engines
# ---------------------------------------------------------------------------

def _check_inputs(signal: Signal, filters: FilterSet, seg_plan: SegmentPlan):
    """Validation in the reference's order (ols.py:232-254)."""
    if signal.domain != "time":
        raise DomainMismatch("convolution needs a time-domain signal")
    if signal.length != seg_plan.signal_len:
        raise PlanMismatch(
            f"signal length {signal.length} != plan {seg_plan.signal_len}")
    if filters.tap_length != seg_plan.tap_len:
        raise PlanMismatch(
            f"filter tap length {filters.tap_length} != plan "
            f"{seg_plan.tap_len}")
    if filters.origin != seg_plan.origin:
        raise PlanMismatch(
            f"filter origin {filters.origin} != plan {seg_plan.origin}")
    if seg_plan.mode == "r2r":
        if signal.value_kind != "real" or filters.value_kind != "real":
            raise PlanMismatch("r2r mode needs real signal and filters")
    else:
        if signal.value_kind != "complex":
            raise PlanMismatch("c2c mode needs a complex signal")
    sig_single = signal.samples.dtype in (torch.float32, torch.complex64)
    fil_single = filters.taps.dtype in (torch.float32, torch.complex64)
    if sig_single != fil_single:
        raise PlanMismatch("signal and filters must share one precision")


def convolve(signal: Signal, filters: FilterSet, seg_plan: SegmentPlan,
             variant: str = "fused", postproc: Optional[PostProcSpec] = None,
             workers: int = 1, out: Optional[torch.Tensor] = None,
             chunk_segments: Optional[int] = None) -> torch.Tensor:
    """Convolve the signal with every filter; returns (n_fil, signal_len)
    (ols.py:257-316).

    Extensions over the reference (all optional):
      out             preallocated result (CUDA, or pinned CPU memory: then
                      the fused engine streams segment chunks host->device->
                      host with copies overlapped with compute);
      chunk_segments  segments per streaming chunk (host path).
    ``workers`` splits the segment range into that many launches; results
    are bit-identical for any value (test_ols.py:242-251).
    """
    pp = postproc if postproc is not None else NONE
    if variant not in ENGINE_VARIANTS:
        raise ValueError(f"variant must be one of {ENGINE_VARIANTS}")
    _check_inputs(signal, filters, seg_plan)
    precision = signal.precision

    if variant == "fused_exact" and (seg_plan.mode != "c2c" or pp.kind not in (
            "none", "scale", "magnitude_squared")):
        raise EngineError("variant 'fused_exact' (the reference's arithmetic) "
                          "covers c2c with postproc none | scale | "
                          "magnitude_squared")
    if pp.kind == "derivative" and variant != "fused":
        # the comparison variants have no segment epilogue: plain result,
        # then the global difference on the device
        plain = convolve(signal, filters, seg_plan, variant, None, workers)
        return _derivative(plain, out)

    if variant in ("direct_oracle", "full_fft_baseline"):
        y = (_direct(signal, filters, pp) if variant == "direct_oracle"
             else full_fft_convolve(signal, filters, pp))
        if out is None:
            return y
        if tuple(out.shape) != tuple(y.shape) or out.dtype != y.dtype:
            raise ValueError(f"out must be {tuple(y.shape)} {y.dtype}")
        out.copy_(y)
        return out

    layout = _required_layout(seg_plan.mode, variant)
    if filters.spectra is None:
        filters = transform_filters(filters, seg_plan, layout)
    else:
        if filters.spectra_n != seg_plan.fft_len:
            raise PlanMismatch(
                f"cached spectra built for length {filters.spectra_n},"
                f" plan wants {seg_plan.fft_len}")
        if filters.spectra_layout != layout:
            raise LayoutMismatch(
                f"cached spectra layout {filters.spectra_layout!r} does not"
                f" match the {variant} engine's transform ({layout!r})")
        want_bins = (seg_plan.fft_len // 2 + 1 if seg_plan.mode == "r2r"
                     else seg_plan.fft_len)
        if filters.spectra.shape[1] != want_bins:
            raise PlanMismatch("cached spectra do not match the plan's mode")

    n_s = signal.length
    n_fil = filters.n_filters
    real_out = seg_plan.mode == "r2r" or pp.real_output
    out_dtype = precision.torch_real if real_out else precision.torch_complex

    if pp.kind == "derivative" and n_s == 1:
        return torch.zeros((n_fil, 1), dtype=out_dtype,
                           device=signal.samples.device)

    l_eff, t0, win_off, n_seg_eff = _geometry(seg_plan, pp.halo)

    if out is not None:
        if tuple(out.shape) != (n_fil, n_s) or out.dtype != out_dtype:
            raise ValueError(f"out must be {(n_fil, n_s)} {out_dtype}")
        if not out.is_contiguous():
            raise ValueError("out must be contiguous")

    if variant == "fused":
        spec_dev = _engine_spectra(filters)
        if out is not None and not out.is_cuda:
            return _fused_streaming(signal, spec_dev, seg_plan, pp, precision,
                                    l_eff, t0, win_off, n_seg_eff, out,
                                    chunk_segments)
        if not signal.samples.is_cuda:
            raise ValueError("a host-resident signal needs a host `out` "
                             "(streaming path)")
        if out is None:
            out = torch.empty((n_fil, n_s), dtype=out_dtype,
                              device=signal.samples.device)
        with torch.cuda.device(signal.samples.device):
            if pp.kind == "derivative" and seg_plan.tap_len == 1:
                # one tap has no aliased region to hold a halo in the
                # reference's geometry (it recomputes seam neighbours from
                # the input, _kernels_nb.py:232-260); the range entries'
                # halo geometry (t0 = 1, L = N - 2) keeps both neighbours in
                # the segment
                for lo, hi in _chunk_bounds(n_s, workers):
                    fused_range_launch(signal.samples, 0, n_s, spec_dev, n_fil,
                                       seg_plan, lo, hi, pp, out, n_s, 0,
                                       precision)
                return out
            for lo, hi in _chunk_bounds(n_seg_eff, workers):
                fused_launch(signal.samples, 0, n_s, spec_dev, n_fil, seg_plan,
                             l_eff, t0, win_off, lo, hi, pp, out, n_s, 0,
                             precision)
        return out
    if variant == "fused_exact":
        return _fused_exact(signal, filters, seg_plan, pp, precision, l_eff,
                            t0, win_off, n_seg_eff, out, out_dtype, workers)
    if variant == "cufft_ols":
        return _cufft_ols(signal, filters, seg_plan, pp, precision,
                                    out)
    return _pipelined(signal, filters, seg_plan, pp, precision, l_eff, t0,
                      win_off, n_seg_eff, out)


_REF_TW = {}


def _ref_twiddles(n: int, precision: Precision, device) -> torch.Tensor:
    """The reference's twiddle table tw[j] = e^{-2 pi i j / n}, j < n/2, as
    fft.py:70-78 builds it (numpy, rounded to the precision), on `device`."""
    key = (n, precision, str(device))
    t = _REF_TW.get(key)
    if t is None:
        from .fft import _tables
        tw = _tables(n, n // 2, precision)[0]
        t = torch.from_numpy(np.array(tw)).to(device)
        _REF_TW[key] = t
    return t


def _fused_exact(signal, filters, seg_plan, pp, precision, l_eff, t0,
                 win_off, n_seg, out, out_dtype, workers):
    """variant="fused_exact": the fused engine with the reference's
    arithmetic (olsb_fused_c2c_ref): outputs bit-identical to the
    reference's fp32 / fp64 ``convolve(variant="fused")``."""
    host_out = out is not None and not out.is_cuda
    if not signal.samples.is_cuda and not host_out:
        raise ValueError("a host-resident signal needs a host `out` "
                         "(streaming path)")
    n, n_s, n_fil = seg_plan.fft_len, signal.length, filters.n_filters
    dev = (signal.samples.device if signal.samples.is_cuda
           else filters.taps.device if filters.taps.is_cuda
           else torch.device("cuda", torch.cuda.current_device()))
    tw = _ref_twiddles(n, precision, dev)
    taps = filters.taps.to(device=dev, dtype=precision.torch_complex)
    taps = taps.contiguous()
    spec = torch.empty((n_fil, n), dtype=precision.torch_complex, device=dev)
    with torch.cuda.device(dev):
        _lib.call("olsb_filter_spectra_c2c_ref", taps.data_ptr(), n_fil,
                  seg_plan.tap_len, n, tw.data_ptr(), None, spec.data_ptr(),
                  precision.code, _stream_ptr())

    def launch(x, f0, f1, dst, ld, stream, lo=0, hi=n_seg):
        if f1 <= f0:
            return
        common = (x.data_ptr(), 0, n_s, spec[f0].data_ptr(), f1 - f0, n,
                  seg_plan.tap_len, seg_plan.origin, l_eff, t0, win_off, lo, hi)
        tail = (dst.data_ptr(), ld, 0, precision.code, stream)
        if pp.kind == "magnitude_squared":
            _lib.call("olsb_fused_c2c_abs2_ref", *common, tw.data_ptr(), *tail)
        else:
            _lib.call("olsb_fused_c2c_ref", *common, pp.code, float(pp.scale),
                      tw.data_ptr(), *tail)

    if host_out:
        # host streaming in chunks of whole output rows (contiguous D2H)
        row = n_s * out.element_size()
        fc = max(1, min(_STREAM_TILE // row, max(1, n_fil // 3)))
        return _fused_streaming_rows(
            signal, spec, seg_plan, pp, precision, out, fc,
            launch=lambda x, f0, f1, ob, st: launch(x, f0, f1, ob, n_s, st))
    if out is None:
        out = torch.empty((n_fil, n_s), dtype=out_dtype, device=dev)
    with torch.cuda.device(dev):
        for lo, hi in _chunk_bounds(n_seg, workers):
            launch(signal.samples, 0, n_fil, out, n_s, _stream_ptr(), lo, hi)
    return out


def _engine_entry(seg_plan: SegmentPlan, pp: PostProcSpec) -> str:
    """C-ABI entry of the fused engine for a plan + post-process: the
    reference's K.fused_c2c / K.fused_c2c_abs2 / K.fused_r2r
    (_kernels_nb.py:265-337)."""
    if seg_plan.mode == "r2r":
        return "olsb_fused_r2r"
    if pp.kind == "magnitude_squared":
        return "olsb_fused_c2c_abs2"
    return "olsb_fused_c2c"


def fused_launch(x: torch.Tensor, x_base: int, n_s: int,
                 spec_dev: torch.Tensor, n_fil: int, seg_plan: SegmentPlan,
                 l_eff: int, t0: int, win_off: int, seg_lo: int, seg_hi: int,
                 pp: PostProcSpec, out: torch.Tensor, out_ld: int,
                 out_base: int, precision: Precision,
                 stream: Optional[int] = None) -> None:
    """One call of the C-ABI fused kernel (the reference's K.fused_c2c,
    K.fused_c2c_abs2 or K.fused_r2r, _kernels_nb.py:265-337) on the current
    stream."""
    entry = _engine_entry(seg_plan, pp)
    common = (x.data_ptr(), x_base, n_s, spec_dev.data_ptr(), n_fil,
              seg_plan.fft_len, seg_plan.tap_len, seg_plan.origin, l_eff, t0,
              win_off, seg_lo, seg_hi)
    tail = (out.data_ptr(), out_ld, out_base, precision.code,
            _stream_ptr() if stream is None else stream)
    if entry == "olsb_fused_c2c_abs2":
        _lib.call(entry, *common, *tail)
    else:
        _lib.call(entry, *common, pp.code, float(pp.scale), *tail)


def fused_range_launch(x: torch.Tensor, x_base: int, n_s: int,
                       spec_dev: torch.Tensor, n_fil: int,
                       seg_plan: SegmentPlan, g_lo: int, g_hi: int,
                       pp: PostProcSpec, out: torch.Tensor, out_ld: int,
                       out_base: int, precision: Precision,
                       stream: Optional[int] = None) -> None:
    """Outputs [g_lo, g_hi) through olsb_fused_{c2c,r2r}_range (shards,
    streams).  Every post-process; the derivative runs in the halo geometry
    (t0 = M, L = N - M - 1), whose input extent input_extent(..., pp)
    gives."""
    entry = ("olsb_fused_r2r_range" if seg_plan.mode == "r2r"
             else "olsb_fused_c2c_range")
    if pp.kind == "derivative" and seg_plan.fft_len - seg_plan.tap_len - 1 < 1:
        raise HaloUnavailable(
            f"segment length {seg_plan.fft_len} leaves no room for a halo of 1"
            f" around {seg_plan.tap_len} taps")
    _lib.call(entry, x.data_ptr(), x_base, n_s, spec_dev.data_ptr(), n_fil,
              seg_plan.fft_len, seg_plan.tap_len, seg_plan.origin, g_lo, g_hi,
              pp.code, float(pp.scale), out.data_ptr(), out_ld, out_base,
              precision.code, _stream_ptr() if stream is None else stream)


def input_extent(seg_plan: SegmentPlan, g_lo: int, g_hi: int,
                 postproc: PostProcSpec = NONE) -> Tuple[int, int]:
    """Input samples [x_lo, x_hi) the engine's range entry reads to produce
    outputs [g_lo, g_hi) with post-process `postproc` (its shard plus halos;
    clip to [0, n_s) before copying)."""
    import ctypes
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.load().olsb_input_extent_pp(
        1 if seg_plan.mode == "r2r" else 0, seg_plan.fft_len,
        seg_plan.tap_len, seg_plan.origin, postproc.code, g_lo, g_hi,
        ctypes.byref(lo), ctypes.byref(hi)), "olsb_input_extent_pp")
    return lo.value, hi.value


_STREAM_TILE = 256 << 20   # bytes of output per streaming chunk


def _fused_streaming(signal, spec_dev, seg_plan, pp, precision, l_eff, t0,
                     win_off, n_seg, out, chunk_segments):
    """Host-memory path: per chunk of outputs, fused kernel into a device
    staging tile and D2H into ``out``.  Three streams rotate over three
    staging slots so copies in both directions overlap the kernel of the
    neighbouring chunks.  When one output row fits a tile and there are at
    least three filters, chunks are blocks of whole rows (filters): every D2H
    is one contiguous copy (~55 GB/s over PCIe against ~51 GB/s for the
    strided copies of segment chunks) and the signal goes to the device once.
    Otherwise (or with ``chunk_segments``) chunks are segment ranges with
    their input extents copied per chunk.  Results are bit-identical either
    way."""
    n_s = signal.length
    n_fil = spec_dev.shape[0]
    esize = out.element_size()
    row = n_s * esize
    if chunk_segments is None and n_fil >= 3 and row <= _STREAM_TILE:
        fc = max(1, min(_STREAM_TILE // row, n_fil // 3))
        return _fused_streaming_rows(signal, spec_dev, seg_plan, pp, precision,
                                     out, fc)
    x_host = signal.samples
    dev = spec_dev.device
    if chunk_segments is None:
        # ~256 MiB of output per chunk
        chunk_segments = max(1, (256 << 20) // max(1, n_fil * l_eff * esize))
    w = max(32, (chunk_segments * l_eff) // 32 * 32)
    chunks = [(g, min(g + w, n_s)) for g in range(0, n_s, w)]
    nslot = min(3, len(chunks))
    ext = [input_extent(seg_plan, ga, gb, pp) for ga, gb in chunks]
    x_len_max = max(min(hi, n_s) - max(lo, 0) for lo, hi in ext)
    with torch.cuda.device(dev):
        streams = [torch.cuda.Stream() for _ in range(nslot)]
        xbuf = [torch.empty(max(1, x_len_max), dtype=x_host.dtype, device=dev)
                for _ in range(nslot)]
        obuf = [torch.empty((n_fil, w), dtype=out.dtype, device=dev)
                for _ in range(nslot)]
        ready = torch.cuda.current_stream()
        for s in streams:
            s.wait_stream(ready)
        lib = _lib.load()
        for i, ((ga, gb), (lo, hi)) in enumerate(zip(chunks, ext)):
            k = i % nslot
            st = streams[k]
            xa, xb = max(0, lo), min(n_s, hi)
            with torch.cuda.stream(st):
                if xb > xa:
                    xbuf[k][:xb - xa].copy_(x_host[xa:xb], non_blocking=True)
                fused_range_launch(xbuf[k], xa, n_s, spec_dev, n_fil, seg_plan,
                                   ga, gb, pp, obuf[k], w, ga, precision,
                                   st.cuda_stream)
                _lib.check(lib.olsb_copy2d_async(
                    out.data_ptr() + ga * esize, n_s * esize,
                    obuf[k].data_ptr(), w * esize, (gb - ga) * esize,
                    n_fil, 0, st.cuda_stream), "olsb_copy2d_async")
        for s in streams:
            ready.wait_stream(s)
        # keep the staging buffers alive until the copies retire
        for s in streams:
            s.synchronize()
    return out


def _fused_streaming_rows(signal, spec_dev, seg_plan, pp, precision, out,
                          fc, launch=None):
    """Host-memory path chunked by filters (see _fused_streaming).
    ``launch(x_dev, f0, f1, obuf, stream)`` replaces the default range
    launch (exact mode)."""
    n_s = signal.length
    n_fil = spec_dev.shape[0]
    dev = spec_dev.device
    chunks = [(f, min(f + fc, n_fil)) for f in range(0, n_fil, fc)]
    nslot = min(3, len(chunks))
    with torch.cuda.device(dev):
        streams = [torch.cuda.Stream() for _ in range(nslot)]
        ready = torch.cuda.current_stream()
        for s in streams:
            s.wait_stream(ready)
        xdev = torch.empty(n_s, dtype=signal.samples.dtype, device=dev)
        with torch.cuda.stream(streams[0]):
            xdev.copy_(signal.samples, non_blocking=True)
        staged = torch.cuda.Event()
        staged.record(streams[0])
        for s in streams[1:]:
            s.wait_event(staged)
        obuf = [torch.empty((fc, n_s), dtype=out.dtype, device=dev)
                for _ in range(nslot)]
        for i, (f0, f1) in enumerate(chunks):
            k = i % nslot
            st = streams[k]
            with torch.cuda.stream(st):
                if launch is not None:
                    launch(xdev, f0, f1, obuf[k], st.cuda_stream)
                else:
                    fused_range_launch(xdev, 0, n_s, spec_dev[f0:f1], f1 - f0,
                                       seg_plan, 0, n_s, pp, obuf[k], n_s, 0,
                                       precision, st.cuda_stream)
                out[f0:f1].copy_(obuf[k][:f1 - f0], non_blocking=True)
        for s in streams:
            ready.wait_stream(s)
        # keep the staging buffers alive until the copies retire
        for s in streams:
            s.synchronize()
    return out


def _derivative(y: torch.Tensor, out: Optional[torch.Tensor] = None):
    """Global central difference with one-sided ends (postproc.py:44-85 with
    both ends flagged as signal edges): d[g] = (y[g+1] - y[g-1]) / 2, d[0] =
    y[1] - y[0], d[-1] = y[-1] - y[-2]."""
    n_s = y.shape[1]
    d = torch.empty_like(y)
    if n_s == 1:
        d.zero_()
    else:
        d[:, 1:n_s - 1] = 0.5 * (y[:, 2:] - y[:, :n_s - 2])
        d[:, 0] = y[:, 1] - y[:, 0]
        d[:, n_s - 1] = y[:, n_s - 1] - y[:, n_s - 2]
    if out is not None:
        out.copy_(d)
        return out
    return d


def _pipelined(signal, filters, seg_plan, pp, precision, l_eff, t0, win_off,
               n_seg, out):
    """cuFFT-based OLS, the paper's comparison point (Algorithm 1;
    reference _pipelined ols.py:363-410): gather -> batched forward FFT (C2C,
    or R2C on the real path) -> materialized product -> batched inverse (C2C /
    C2R) -> discard + store.  Chunked so the (n_fil, rows, n) product stays
    within PIPELINED_BUDGET_BYTES."""
    n = seg_plan.fft_len
    n_s = signal.length
    x = signal.samples
    spectra = filters.spectra  # natural order (rfft bins on the real path)
    n_fil = filters.n_filters
    dev = x.device
    real = seg_plan.mode == "r2r"
    real_out = real or pp.real_output
    if out is None:
        out = torch.empty((n_fil, n_s), dtype=(precision.torch_real if real_out
                                               else precision.torch_complex),
                          device=dev)
    csize = 8 if precision == Precision.single else 16
    rows_per = max(1, PIPELINED_BUDGET_BYTES // (2 * n_fil * n * csize))
    ar = torch.arange(n, device=dev)
    for lo in range(0, n_seg, rows_per):
        hi = min(lo + rows_per, n_seg)
        starts = torch.arange(lo, hi, device=dev) * l_eff + win_off
        idx = starts[:, None] + ar[None, :]
        ok = (idx >= 0) & (idx < n_s)
        mat = torch.where(ok, x[idx.clamp(0, n_s - 1)],
                          torch.zeros((), dtype=x.dtype, device=dev))
        if real:
            fmat = torch.fft.rfft(mat, dim=1)
            mid = torch.fft.irfft(fmat[None, :, :] * spectra[:, None, :], n=n,
                                  dim=2)
        else:
            fmat = torch.fft.fft(mat, dim=1)
            mid = torch.fft.ifft(fmat[None, :, :] * spectra[:, None, :], dim=2)
        valid = mid[:, :, t0:t0 + l_eff].reshape(n_fil, -1)
        g_lo = lo * l_eff
        g_hi = min(hi * l_eff, n_s)
        seg_out = valid[:, :g_hi - g_lo]
        if pp.kind == "scale":
            seg_out = seg_out * pp.scale
        elif pp.kind == "magnitude_squared":
            seg_out = (seg_out * seg_out if real else
                       seg_out.real * seg_out.real + seg_out.imag * seg_out.imag)
        out[:, g_lo:g_hi] = seg_out
    return out


def _cufft_ols(signal, filters, seg_plan, pp, precision, out):
    """The paper's cuFFT-OLS in its efficient form (Algorithm 1;
    libolsb_cufft.so, csrc/olsb_cufft.cu): per L2-sized chunk of segments a
    batched forward C2C that reads the overlapping windows in place (idist =
    L), then per chunk of filters a multiply kernel, one batched inverse C2C
    and a store kernel that keeps only the valid samples.  (The paper puts
    the multiply and the discard into cuFFT callbacks; on this platform
    cuFFT does not apply them, see csrc/olsb_cufft.cu.)  c2c, single
    precision, postproc none / scale."""
    from . import _lib_cufft
    if (seg_plan.mode != "c2c" or precision != Precision.single
            or pp.kind not in ("none", "scale")):
        raise EngineError("variant 'cufft_ols' covers c2c, single "
                          "precision, postproc none | scale")
    x = signal.samples
    if not x.is_cuda:
        raise ValueError("variant 'cufft_ols' needs a device signal")
    n, n_s, n_fil = seg_plan.fft_len, signal.length, filters.n_filters
    if out is None:
        out = torch.empty((n_fil, n_s), dtype=torch.complex64, device=x.device)
    spec = filters.spectra.to(device=x.device, dtype=torch.complex64).contiguous()
    with torch.cuda.device(x.device):
        _lib_cufft.ols_c2c(x, n_s, spec, n_fil, n, seg_plan.tap_len,
                           seg_plan.origin, out, n_s, _stream_ptr())
    if pp.kind == "scale":
        out.mul_(pp.scale)
    return out


def _direct(signal: Signal, filters: FilterSet, pp: PostProcSpec):
    """Direct time-domain convolution on the GPU, float64 accumulate, rounded
    to the signal's precision (oracle.py:20-41): y[f,n] = sum_k h[f,k]
    x[n-k+o], zeros off the ends.  Complex conv = 4 real conv1d calls."""
    real = signal.value_kind == "real" and filters.value_kind == "real"
    x = signal.samples.to(torch.complex128)
    h = filters.taps.to(torch.complex128)
    m = filters.tap_length
    o = filters.origin
    n_s = signal.length
    # cross-correlation with flipped taps == convolution
    hf = torch.flip(h, dims=[1])
    pad_l, pad_r = m - 1 - o, o
    xr = torch.nn.functional.pad(x.real[None, None], (pad_l, pad_r))
    xi = torch.nn.functional.pad(x.imag[None, None], (pad_l, pad_r))
    wr = hf.real[:, None, :].contiguous()
    wi = hf.imag[:, None, :].contiguous()
    conv = torch.nn.functional.conv1d
    yr = conv(xr, wr)[0] - conv(xi, wi)[0]
    yi = conv(xr, wi)[0] + conv(xi, wr)[0]
    y = torch.complex(yr, yi)[:, :n_s]
    if pp.kind == "scale":
        y = y * pp.scale
    if real:
        y = y.real
        if pp.kind == "magnitude_squared":
            y = y * y
        return y.to(signal.precision.torch_real)
    if pp.kind == "magnitude_squared":
        return (y.real * y.real + y.imag * y.imag).to(
            signal.precision.torch_real)
    return y.to(signal.precision.torch_complex)


def full_fft_convolve(signal: Signal, filters: FilterSet,
                      postproc: Optional[PostProcSpec] = None,
                      max_len: int = DEFAULT_MAX_FULL_LEN) -> torch.Tensor:
    """No-segmentation baseline (ols.py:413-464): one cuFFT convolution of the
    whole signal padded to next_pow2(n_s + m - 1)."""
    pp = postproc if postproc is not None else NONE
    if signal.domain != "time":
        raise DomainMismatch("convolution needs a time-domain signal")
    if signal.value_kind == "real" and filters.value_kind == "complex":
        raise PlanMismatch("complex filter taps on a real signal")
    if pp.kind not in ("none", "scale"):
        raise EngineError("full_fft_convolve supports postproc none|scale only")
    precision = signal.precision
    n_s = signal.length
    m = filters.tap_length
    o = filters.origin
    real_path = signal.value_kind == "real"
    padded_len = max(8 if real_path else 4, next_pow2(n_s + m - 1))
    if padded_len > max_len:
        raise TooLarge(
            f"padded length {padded_len} exceeds the {max_len}-sample budget")
    x = signal.samples
    h = filters.taps
    if real_path:
        full = torch.fft.irfft(torch.fft.rfft(x, n=padded_len)[None, :]
                               * torch.fft.rfft(h, n=padded_len, dim=1),
                               n=padded_len, dim=1)
    else:
        h = h.to(precision.torch_complex)
        full = torch.fft.ifft(torch.fft.fft(x, n=padded_len)[None, :]
                              * torch.fft.fft(h, n=padded_len, dim=1), dim=1)
    y = full[:, o:o + n_s]
    if pp.kind == "scale":
        y = y * pp.scale
    return y.contiguous()


# ---------------------------------------------------------------------------
# segment-size autotuning (ols.py:471-526), timed with CUDA events
# ---------------------------------------------------------------------------

def measure_segment_times(tap_len: int, mode: str, candidates: Iterable[int],
                          probe_len: int = 1 << 18, n_filters: int = 4,
                          repeats: int = 3,
                          precision: Precision = Precision.single,
                          seed: int = 0) -> dict:
    """Median fused-engine device time per feasible candidate length."""
    floor = 8 if mode == "r2r" else 4
    feasible = sorted(c for c in set(candidates)
                      if _is_pow2(c) and c >= max(tap_len, floor))
    if not feasible:
        raise SegmentTooSmall(
            f"no candidate segment length fits {tap_len} taps")
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    rng = np.random.default_rng(seed)
    if mode == "r2r":
        sig = make_signal(rng.standard_normal(probe_len), "real", precision)
        taps = rng.standard_normal((n_filters, tap_len))
    else:
        sig = make_signal(rng.standard_normal(probe_len)
                          + 1j * rng.standard_normal(probe_len), "complex",
                          precision)
        taps = (rng.standard_normal((n_filters, tap_len))
                + 1j * rng.standard_normal((n_filters, tap_len)))
    fs = make_filterset(taps, 0, precision)
    times = {}
    for cand in feasible:
        p = plan(probe_len, tap_len, mode, 0, cand,
                 max_fft_len=max(cand, DEFAULT_MAX_FFT_LEN))
        if cand > DEFAULT_MAX_FFT_LEN:
            continue
        cached = transform_filters(fs, p, _required_layout(mode, "fused"))
        out = convolve(sig, cached, p)
        samples = []
        for _ in range(repeats):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            convolve(sig, cached, p, out=out)
            e1.record()
            e1.synchronize()
            samples.append(e0.elapsed_time(e1) * 1e-3)
        times[cand] = float(np.median(samples))
    return times


def autotune_segment_size(tap_len: int, mode: str,
                          candidates: Optional[Iterable[int]] = None,
                          probe_len: int = 1 << 18, **kwargs) -> int:
    """Fastest candidate; ties go to the smaller length (ols.py:511-526)."""
    if candidates is None:
        candidates = [1 << b for b in range(6, 13)]
    times = measure_segment_times(tap_len, mode, candidates, probe_len,
                                  **kwargs)
    best_n, best_t = None, math.inf
    for cand in sorted(times):
        if times[cand] < best_t:
            best_n, best_t = cand, times[cand]
    return best_n
