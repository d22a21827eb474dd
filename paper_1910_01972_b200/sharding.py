"""Multi-GPU signal partitioning.

The long signal is split across ranks as contiguous output ranges on the
reference's segment grid (ols._chunk_bounds, ols.py:212-215).  Rank r owns
outputs [g_lo, g_hi) and the matching input samples; to compute its outputs
it also needs a few samples on each side (the (M-1)-sample overlap of its
first and last segment windows), fetched from its neighbours with one
point-to-point exchange (NCCL send/recv over NVLink on B200; gloo on CPU).
There is no collective on the hot path and the outputs stay sharded.

Because the engine's segment grid is anchored at global sample 0
(olsb_fused_c2c_range), every output sample is computed by the same segment
whatever the partition, so sharded results are bit-identical to a
single-GPU run.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

import torch
import torch.distributed as dist

from .ols import SegmentPlan, _chunk_bounds, input_extent


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    g_lo: int        # owned outputs [g_lo, g_hi) == owned input samples
    g_hi: int
    x_lo: int        # input samples the engine reads, clipped to [0, n_s)
    x_hi: int

    @property
    def left_halo(self) -> int:
        return self.g_lo - self.x_lo

    @property
    def right_halo(self) -> int:
        return self.x_hi - self.g_hi


def shard_bounds(n_seg: int, valid_len: int, n_s: int, world: int) -> List[Tuple[int, int]]:
    """Owned output ranges per rank: contiguous reference segments."""
    out = []
    for lo, hi in _chunk_bounds(n_seg, world):
        out.append((lo * valid_len, min(hi * valid_len, n_s)))
    while len(out) < world:          # more ranks than segments: empty shards
        out.append((n_s, n_s))
    return out


def make_shards(seg_plan: SegmentPlan, world: int, extent=None,
                postproc=None) -> List[Shard]:
    """Shard layout for every rank.  ``extent(g_lo, g_hi) -> (x_lo, x_hi)``
    defaults to the engine's input extent for post-process ``postproc``
    (olsb_input_extent_pp: the derivative's halo geometry reads one more
    segment of context than the plain one)."""
    from .postproc import NONE
    pp = postproc or NONE
    extent = extent or (lambda a, b: input_extent(seg_plan, a, b, pp))
    n_s = seg_plan.signal_len
    shards = []
    for r, (g_lo, g_hi) in enumerate(shard_bounds(seg_plan.n_segments,
                                                  seg_plan.valid_len, n_s,
                                                  world)):
        if g_hi > g_lo:
            x_lo, x_hi = extent(g_lo, g_hi)
            x_lo, x_hi = max(0, x_lo), min(n_s, x_hi)
        else:
            x_lo = x_hi = g_lo
        shards.append(Shard(r, world, g_lo, g_hi, min(x_lo, g_lo),
                            max(x_hi, g_hi)))
    return shards


def exchange_halos(own: torch.Tensor, shards: List[Shard], rank: int,
                   group=None) -> torch.Tensor:
    """Assemble rank `rank`'s engine input [x_lo, x_hi) from its owned
    samples [g_lo, g_hi) plus halos received from the neighbours.

    Every rank sends the parts of its owned range that other ranks' extents
    cover (normally only the two neighbours) with one batched P2P exchange.
    Works with any torch.distributed backend (NCCL on GPUs, gloo on CPU).
    """
    me = shards[rank]
    buf = torch.empty(me.x_hi - me.x_lo, dtype=own.dtype, device=own.device)
    buf[me.g_lo - me.x_lo:me.g_hi - me.x_lo] = own
    ops = []
    recvs = []
    for peer in shards:
        if peer.rank == rank:
            continue
        # what I need from peer: overlap of my extent with peer's ownership
        lo, hi = max(me.x_lo, peer.g_lo), min(me.x_hi, peer.g_hi)
        if hi > lo:
            view = buf[lo - me.x_lo:hi - me.x_lo]
            tmp = torch.empty_like(view)
            ops.append(dist.P2POp(dist.irecv, tmp, peer.rank, group))
            recvs.append((view, tmp))
        # what peer needs from me
        lo, hi = max(peer.x_lo, me.g_lo), min(peer.x_hi, me.g_hi)
        if hi > lo:
            ops.append(dist.P2POp(dist.isend,
                                  own[lo - me.g_lo:hi - me.g_lo].contiguous(),
                                  peer.rank, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for view, tmp in recvs:
        view.copy_(tmp)
    return buf


class HaloBuffer:
    """Persistent halo'd input of one rank: ``buffer`` holds input samples
    [x_lo, x_hi); the rank writes its owned samples into ``own`` (the view
    [g_lo, g_hi)) once, and every step :meth:`exchange` moves ONLY the halos
    -- the (M-1-o) samples left and o right of the shard, each from the
    neighbour that owns them -- by one batched NCCL send/recv (NVLink P2P on
    B200; gloo on CPU).  No allocation and no copy of the owned range per
    step, no collective.
    """

    def __init__(self, shards: List[Shard], rank: int, dtype, device,
                 group=None):
        self.shards = shards
        self.rank = rank
        self.group = group
        me = shards[rank]
        self.shard = me
        self.buffer = torch.zeros(max(1, me.x_hi - me.x_lo), dtype=dtype,
                                  device=device)
        self.own = self.buffer[me.g_lo - me.x_lo:me.g_hi - me.x_lo]
        # (peer, recv view of my buffer) / (peer, send view of my own range)
        self.recvs, self.sends = [], []
        for peer in shards:
            if peer.rank == rank:
                continue
            lo, hi = max(me.x_lo, peer.g_lo), min(me.x_hi, peer.g_hi)
            if hi > lo:
                self.recvs.append((peer.rank,
                                   self.buffer[lo - me.x_lo:hi - me.x_lo]))
            lo, hi = max(peer.x_lo, me.g_lo), min(peer.x_hi, me.g_hi)
            if hi > lo:
                self.sends.append((peer.rank,
                                   self.buffer[lo - me.x_lo:hi - me.x_lo]))

    @property
    def halo_samples(self) -> int:
        return sum(v.numel() for _, v in self.recvs)

    def exchange(self) -> torch.Tensor:
        """Receive this step's halos (the neighbours' boundary samples) into
        the buffer; returns the buffer ([x_lo, x_hi))."""
        ops = [dist.P2POp(dist.irecv, v, peer, self.group)
               for peer, v in self.recvs]
        ops += [dist.P2POp(dist.isend, v, peer, self.group)
                for peer, v in self.sends]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return self.buffer

    def fill_from(self, x_global: torch.Tensor) -> torch.Tensor:
        """Single-process emulation of :meth:`exchange` (one GPU standing in
        for several ranks): the halos are device copies out of the global
        signal instead of P2P receives."""
        for peer, v in self.recvs:
            off = self.shard.x_lo + (v.data_ptr() - self.buffer.data_ptr()) // v.element_size()
            v.copy_(x_global[off:off + v.numel()])
        return self.buffer


def convolve_shard_chunked(x_local: torch.Tensor, shard: Shard,
                           seg_plan: SegmentPlan, spec_dev: torch.Tensor,
                           n_fil: int, precision, out_chunk: torch.Tensor,
                           sink=None, stream: Optional[int] = None) -> int:
    """This rank's outputs [g_lo, g_hi) in passes of ``out_chunk.shape[1]``
    outputs per filter into the reused device tile ``out_chunk`` (n_fil x
    w): the per-rank output can exceed HBM (cfg5 at 2 GPUs: 256 GiB per
    rank).  ``sink(g_a, g_b, tile)`` consumes each pass (copy out, reduce,
    or nothing when only the device throughput is measured).  Pass
    boundaries are multiples of the engine's segment grid only for
    efficiency; any cut is bit-identical (the grid is anchored at sample 0).
    Returns the number of launches."""
    from .postproc import NONE
    from .ols import fused_range_launch
    w = out_chunk.shape[1]
    launches = 0
    for g_a in range(shard.g_lo, shard.g_hi, w):
        g_b = min(g_a + w, shard.g_hi)
        fused_range_launch(x_local, shard.x_lo, seg_plan.signal_len, spec_dev,
                           n_fil, seg_plan, g_a, g_b, NONE, out_chunk, w, g_a,
                           precision, stream)
        launches += 1
        if sink is not None:
            sink(g_a, g_b, out_chunk)
    return launches


def convolve_shard(x_local: torch.Tensor, shard: Shard, seg_plan: SegmentPlan,
                   filters, out: Optional[torch.Tensor] = None,
                   postproc=None) -> torch.Tensor:
    """This rank's outputs [g_lo, g_hi) of every filter from its halo'd input
    (x_local covers [x_lo, x_hi)); one fused-engine launch."""
    from .ols import _engine_spectra, fused_range_launch, transform_filters
    from .postproc import NONE
    pp = postproc or NONE
    if filters.spectra is None:
        filters = transform_filters(
            filters, seg_plan, "natural" if seg_plan.mode == "r2r" else "permuted")
    spec = _engine_spectra(filters)
    width = shard.g_hi - shard.g_lo
    if out is None:
        out = torch.empty((filters.n_filters, width), dtype=x_local.dtype,
                          device=x_local.device)
    if width > 0:
        prec = (filters.taps.dtype in (torch.float32, torch.complex64))
        from .core import Precision
        fused_range_launch(x_local, shard.x_lo, seg_plan.signal_len, spec,
                           filters.n_filters, seg_plan, shard.g_lo, shard.g_hi,
                           pp, out, width, shard.g_lo,
                           Precision.single if prec else Precision.double)
    return out
