"""Bound convolution executor: the fused engine with everything but the data
pointers prepared once.

``convolve`` (ols.py) re-validates its arguments and rebuilds the launch on
every call, which costs ~20 us of host time -- the whole budget of a small
cell (cfg1: 2^20 samples, one filter).  An ``Executor`` binds a plan, a filter
bank and a post-process once; each call then checks shapes and issues one
C-ABI launch.  ``graph()`` captures the launch for fixed buffers into a CUDA
graph, so a replay costs one graph launch.

Results are bit-identical to ``convolve(..., variant="fused")``.

    ex = Executor(filters, seg_plan)
    y = ex(signal)                       # like convolve(signal, filters, plan)
    run = ex.graph(x_tensor, out)        # fixed buffers
    run()                                # replays the captured launch
"""

from __future__ import annotations

from typing import Callable, Optional

import torch

from . import _lib
from .core import FilterSet, Precision, Signal
from .errors import EngineError, PlanMismatch
from .ols import (SegmentPlan, _engine_entry, _engine_spectra, _geometry,
                  _required_layout, _stream_ptr, transform_filters)
from .postproc import NONE, PostProcSpec


class Executor:
    """The fused engine bound to (filters, plan, postproc)."""

    def __init__(self, filters: FilterSet, seg_plan: SegmentPlan,
                 postproc: Optional[PostProcSpec] = None):
        pp = postproc if postproc is not None else NONE
        if filters.tap_length != seg_plan.tap_len:
            raise PlanMismatch(
                f"filter tap length {filters.tap_length} != plan "
                f"{seg_plan.tap_len}")
        if filters.origin != seg_plan.origin:
            raise PlanMismatch(
                f"filter origin {filters.origin} != plan {seg_plan.origin}")
        if seg_plan.mode == "r2r" and filters.value_kind != "real":
            raise PlanMismatch("complex filter taps on the real path")
        layout = _required_layout(seg_plan.mode, "fused")
        if filters.spectra is None or filters.spectra_n != seg_plan.fft_len:
            filters = transform_filters(filters, seg_plan, layout)
        self.filters = filters
        self.plan = seg_plan
        self.postproc = pp
        self.precision = (Precision.single
                          if filters.taps.dtype in (torch.float32,
                                                    torch.complex64)
                          else Precision.double)
        self.spec_dev = _engine_spectra(filters)
        self.device = self.spec_dev.device
        self.n_fil = filters.n_filters
        l_eff, t0, win_off, n_seg = _geometry(seg_plan, pp.halo)
        if pp.kind == "derivative" and seg_plan.tap_len == 1:
            # one tap: the range entry's halo geometry (as convolve())
            name = ("olsb_fused_r2r_range" if seg_plan.mode == "r2r"
                    else "olsb_fused_c2c_range")
            self._entry = getattr(_lib.load(), name)
            self._abs2 = False
            self._head = (seg_plan.signal_len, self.spec_dev.data_ptr(),
                          self.n_fil, seg_plan.fft_len, seg_plan.tap_len,
                          seg_plan.origin, 0, seg_plan.signal_len)
        else:
            self._entry = getattr(_lib.load(), _engine_entry(seg_plan, pp))
            self._abs2 = _engine_entry(seg_plan, pp) == "olsb_fused_c2c_abs2"
            self._head = (seg_plan.signal_len, self.spec_dev.data_ptr(),
                          self.n_fil, seg_plan.fft_len, seg_plan.tap_len,
                          seg_plan.origin, l_eff, t0, win_off, 0, n_seg)
        self._pp = () if self._abs2 else (pp.code, float(pp.scale))
        real_in = seg_plan.mode == "r2r"
        real_out = real_in or pp.real_output
        p = self.precision
        self.in_dtype = p.torch_real if real_in else p.torch_complex
        self.out_dtype = p.torch_real if real_out else p.torch_complex

    def _check(self, x: torch.Tensor, out: torch.Tensor) -> None:
        n_s = self.plan.signal_len
        if x.dtype != self.in_dtype or x.numel() != n_s or not x.is_contiguous():
            raise ValueError(f"signal must be a contiguous {self.in_dtype} "
                             f"tensor of {n_s} samples")
        if (tuple(out.shape) != (self.n_fil, n_s) or out.dtype != self.out_dtype
                or not out.is_contiguous()):
            raise ValueError(f"out must be a contiguous {(self.n_fil, n_s)} "
                             f"{self.out_dtype} tensor")
        if x.device != self.device or out.device != self.device:
            raise ValueError(f"signal and out must live on {self.device}")

    def launch(self, x: torch.Tensor, out: torch.Tensor,
               stream: Optional[int] = None) -> None:
        """One engine launch on `stream` (default: the current stream); no
        validation beyond what the C ABI does."""
        rc = self._entry(x.data_ptr(), 0, *self._head, *self._pp,
                         out.data_ptr(), self.plan.signal_len, 0,
                         self.precision.code,
                         _stream_ptr() if stream is None else stream)
        if rc:
            _lib.check(rc, "fused launch")

    def __call__(self, signal, out: Optional[torch.Tensor] = None
                 ) -> torch.Tensor:
        x = signal.samples if isinstance(signal, Signal) else signal
        if out is None:
            out = torch.empty((self.n_fil, self.plan.signal_len),
                              dtype=self.out_dtype, device=self.device)
        self._check(x, out)
        with torch.cuda.device(self.device):
            self.launch(x, out)
        return out

    def graph(self, x: torch.Tensor, out: torch.Tensor,
              launches: int = 1) -> Callable[[], None]:
        """Capture `launches` back-to-back launches for these buffers into a
        CUDA graph; returns a replay function (updating `x` in place and
        replaying re-runs the convolution)."""
        self._check(x, out)
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream(device=self.device)
        with torch.cuda.device(self.device):
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                self.launch(x, out, st.cuda_stream)   # warm-up outside capture
                st.synchronize()
                with torch.cuda.graph(g, stream=st):
                    for _ in range(launches):
                        self.launch(x, out, st.cuda_stream)
            torch.cuda.current_stream().wait_stream(st)

        def replay() -> None:
            g.replay()
        replay.graph = g
        return replay
