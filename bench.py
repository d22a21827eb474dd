"""Benchmark of the fused OLS engine (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

Workload: BASELINE config 3, the FDAS-like filter bank named by north_star's
70%-of-HBM target: 2^23 complex fp32 samples per GPU, 96 filters of 400
taps, FFT segment N = 2048 (weak scaling: the global signal is N_gpus x 2^23
samples, sharded contiguously with (M-1)-sample halos exchanged by NCCL
send/recv inside every step).  A step = halo exchange + one fused-kernel
launch producing every output of the rank's shard (filter spectra are
precomputed and excluded, as in the reference bench, cli.py:229-233).
Inputs: the reference generator convention (cli.py:41-55), synthetic.

Prints ONE JSON line on rank 0.  ``value`` is device-resident throughput
(output samples/s over all ranks, max-over-ranks device time), ``e2e`` the
same metric through the public API from pinned host memory (H2D of the
input, D2H of every output sample, copies overlapped with compute by the
streaming path), ``roofline`` the fused kernel against the measured HBM
bandwidth, ``cpu_baseline`` the oracle's C restatement of the reference on
the host cores.  ``--impl reference`` times that CPU path alone.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

METRIC = ("convolved output samples/s (all filters) and HBM GB/s fraction at "
          "1/2/4/8 B200")
NS, M, NFIL, NFFT = 1 << 23, 400, 96, 2048
WORKLOAD = ("cfg3 FDAS-like filter bank: 2^23 complex fp32 samples per GPU, "
            "96 filters M=400, N=2048")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clock / throttle sampling during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs ~0.1-0.3 s to start: wait for its first
            # sample so the loaded region is actually observed
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5:
                time.sleep(0.01)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


class CpuReference:
    """The reference's CPU path on the host cores: the oracle's C restatement
    of the reference fused kernel (fp32, _kernels_nb.py:265-285, pinned
    bit-exact to the reference's own outputs), split into contiguous segment
    ranges over all host threads like ols.py:212-225.  The sample is the
    FULL cfg3 workload (2^23 samples x 96 filters, N = 2048), timed per call
    like the reference bench times a cell (cli.py:173-181, 223-241)."""

    def __init__(self):
        import oracle
        from cases import gen_inputs
        x, taps = gen_inputs(NS, M, NFIL)
        self.oracle = oracle
        self.x = x.astype(np.complex64)
        self.taps = taps.astype(np.complex64)
        self.threads = oracle.max_threads()
        oracle.fused_convolve(self.x[:1 << 14], self.taps, NFFT, 0, "single",
                              self.threads)

    def run_once(self) -> float:
        t0 = time.perf_counter()
        self.oracle.fused_convolve(self.x, self.taps, NFFT, 0, "single",
                                   self.threads)
        return time.perf_counter() - t0

    def describe(self, secs: float, repeats: int) -> dict:
        return {"value": NS * NFIL / secs, "unit": "samples/s",
                "cores": self.threads, "kind": "port",
                "sample": f"full cfg3 workload: {NS} samples x {NFIL} filters "
                          f"(M={M}, N={NFFT}), median of {repeats}",
                "same_config": True}


def cpu_baseline(repeats: int = 2):
    ref = CpuReference()
    t = statistics.median(ref.run_once() for _ in range(repeats))
    return ref.describe(t, repeats)


def run_reference(args, rank: int):
    """--impl reference: the reference's CPU path (C port of its numba
    kernels, oracle/) on the host cores, same metric and config: every step
    is one full cfg3 convolution."""
    if rank != 0:
        return
    ref = CpuReference()
    for _ in range(args.warmup):
        ref.run_once()
    secs_all = [ref.run_once() for _ in range(args.steps)]
    secs = statistics.median(secs_all)
    cb = ref.describe(secs, args.steps)
    v = cb["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "complex64 (fp32)",
        "data": "synthetic (reference generator convention, cli.py:41-55)",
        "config": {"workload": WORKLOAD, "signal_samples": NS,
                   "filters": NFIL, "taps": M, "fft_len": NFFT,
                   "sample_per_step": cb["sample"],
                   "parallelism": "host threads (pthreads over segments)"},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


CFG5 = dict(ns=1 << 30, m=512, nfil=64, n=4096)
CFG5_TILE = 1 << 26      # outputs per filter per pass (64 x 2^26 x 8 B = 32 GiB)


def run_cfg5(args, world, rank, dev, ob, emulate):
    """BASELINE config 5 (north_star's scaling shape): 2^30 complex samples,
    64 filters M=512, N=4096, halo-sharded over G GPUs (G = the torchrun
    world, or ``emulate`` ranks run one after another on this GPU).  Each
    rank holds its contiguous shard in a persistent halo'd buffer
    (sharding.HaloBuffer) that receives only the (M-1)-sample halos per step
    (NCCL P2P; device copies when emulated) and produces its 2^30/G x 64
    outputs in passes of CFG5_TILE outputs per filter into one reused 32 GiB
    tile (256 GiB per rank at G = 2 does not fit HBM).  Time per rank: CUDA
    events on the rank's stream around halo exchange + every pass; the job
    time is the max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_1910_01972_b200.sharding import (HaloBuffer,
                                                convolve_shard_chunked,
                                                make_shards)
    c = CFG5
    G = emulate or world
    P = ob.Precision.single
    p = ob.plan(c["ns"], c["m"], "c2c", 0, c["n"])
    shards = make_shards(p, G)
    rng = np.random.default_rng([0, c["ns"], c["m"], c["nfil"], 0, 0])
    taps = (rng.standard_normal((c["nfil"], c["m"]))
            + 1j * rng.standard_normal((c["nfil"], c["m"])))
    fs = ob.transform_filters(ob.make_filterset(taps, 0, P, device=dev), p,
                              "permuted")
    spec = fs.spectra_dev
    own_max = max(s.g_hi - s.g_lo for s in shards)
    tile = torch.empty((c["nfil"], min(CFG5_TILE, own_max)),
                       dtype=torch.complex64, device=dev)
    gen = torch.Generator(device=dev)
    steps = max(1, min(args.steps, args.cfg5_steps))

    def time_rank(hb, exchange):
        for _ in range(2):                  # warm-up
            exchange()
            convolve_shard_chunked(hb.buffer, hb.shard, p, spec, c["nfil"], P,
                                   tile)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        passes = 0
        for _ in range(steps):
            exchange()
            passes = convolve_shard_chunked(hb.buffer, hb.shard, p, spec,
                                            c["nfil"], P, tile)
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / steps, passes

    per_rank = []
    if emulate:
        # one global signal; every emulated rank copies its shard into its
        # own halo'd buffer (untimed), then times halo copies + its passes
        xg = torch.randn(c["ns"], dtype=torch.complex64, device=dev,
                         generator=gen.manual_seed(0))
        for r in range(G):
            hb = HaloBuffer(shards, r, torch.complex64, dev)
            sh = shards[r]
            hb.own.copy_(xg[sh.g_lo:sh.g_hi])
            ms, passes = time_rank(hb, lambda hb=hb: hb.fill_from(xg))
            per_rank.append((ms, sh.g_hi - sh.g_lo, passes, hb.halo_samples))
            del hb
        del xg
    else:
        hb = HaloBuffer(shards, rank, torch.complex64, dev)
        sh = shards[rank]
        hb.own.copy_(torch.randn(sh.g_hi - sh.g_lo, dtype=torch.complex64,
                                 device=dev, generator=gen.manual_seed(rank)))
        ms, passes = time_rank(hb, hb.exchange if world > 1 else (lambda: None))
        mine = torch.tensor([ms, sh.g_hi - sh.g_lo, passes, hb.halo_samples],
                            dtype=torch.float64, device=dev)
        if world > 1:
            allv = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(allv, mine)
            per_rank = [tuple(v.tolist()) for v in allv]
        else:
            per_rank = [tuple(mine.tolist())]
    del tile
    torch.cuda.empty_cache()
    hbm, _ = peaks()
    t_max = max(r[0] for r in per_rank)
    fracs = [8 * r[1] * (1 + c["nfil"]) / (r[0] * 1e-3) / 1e9 / hbm
             for r in per_rank]
    return {
        "workload": "cfg5: 2^30 complex fp32 samples, 64 filters M=512, "
                    f"N=4096, halo-sharded over {G} GPU(s)",
        "gpus": G, "emulated": bool(emulate),
        "value": c["ns"] * c["nfil"] / (t_max * 1e-3), "unit": "samples/s",
        "ms_per_step": t_max,
        "per_rank_ms": [round(r[0], 3) for r in per_rank],
        "per_gpu_hbm_frac": [round(f, 4) for f in fracs],
        "passes_per_rank": int(max(r[2] for r in per_rank)),
        "halo_samples_per_rank": [int(r[3]) for r in per_rank],
        "steps": steps,
        "note": ("ranks run one after another on one GPU; halos are device "
                 "copies; value = outputs of all ranks / max rank time"
                 if emulate else
                 "one process per GPU; halos by NCCL P2P; max over ranks"),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cufft", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true")
    ap.add_argument("--cfg5-steps", type=int, default=3)
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="cfg5 leg only: emulate G ranks on this one GPU")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_1910_01972_b200 as ob
    from paper_1910_01972_b200.ols import fused_range_launch
    from paper_1910_01972_b200.sharding import (HaloBuffer,
                                                convolve_shard_chunked,
                                                make_shards)

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)

    P = ob.Precision.single
    ns_global = NS * world
    p = ob.plan(ns_global, M, "c2c", 0, NFFT)
    shards = make_shards(p, world)
    me = shards[rank]
    n_own = me.g_hi - me.g_lo

    # ---- inputs (reference generator convention at N=1)
    from cases import gen_inputs
    if world == 1:
        x_np, taps = gen_inputs(NS, M, NFIL)
    else:
        rng = np.random.default_rng([0, ns_global, M, NFIL, 0, rank + 1])
        x_np = rng.standard_normal(n_own) + 1j * rng.standard_normal(n_own)
        taps = (np.random.default_rng([0, ns_global, M, NFIL, 0, 0])
                .standard_normal((NFIL, M)) * (1 + 1j))
    # the rank's persistent halo'd input: owned samples written once, only
    # the (M-1) halo samples move per step (NCCL P2P)
    hb = HaloBuffer(shards, rank, torch.complex64, dev)
    hb.own.copy_(torch.from_numpy(x_np[me.g_lo:me.g_hi] if world == 1
                                  else x_np).to(dev, torch.complex64))
    fs = ob.transform_filters(ob.make_filterset(taps, 0, P, device=dev), p,
                              "permuted")
    out = torch.empty((NFIL, n_own), dtype=torch.complex64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(ev=None):
        xl = hb.exchange() if world > 1 else hb.buffer
        if ev is not None:
            ev[0].record()
        fused_range_launch(xl, me.x_lo, ns_global, fs.spectra_dev, NFIL, p,
                           me.g_lo, me.g_hi, ob.NONE, out, n_own, me.g_lo, P)
        if ev is not None:
            ev[1].record()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    # clocks are sampled from the warm-up through the timed steps (the timed
    # region alone is ~40 ms, a few nvidia-smi samples)
    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for i in range(args.steps):
            flush.zero_()          # L2 flush between timed steps (untimed)
            starts[i].record()
            step(kev[i])
            ends[i].record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    step_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    kern_ms = [a.elapsed_time(b) for a, b in kev]
    t = torch.tensor([step_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms_max = float(t.item())
    ms_per_step = step_ms_max / args.steps
    outputs_per_step = ns_global * NFIL
    value = outputs_per_step / (ms_per_step * 1e-3)

    hbm, peak_kind = peaks()
    kmean = statistics.mean(kern_ms)
    alg_bytes = 8 * n_own * (1 + NFIL)
    achieved = alg_bytes / (kmean * 1e-3) / 1e9
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic_cfg3.json")
    if os.path.exists(tpath) and world == 1:
        with open(tpath) as f:
            tj = json.load(f)
        traffic = tj.get("dram_bytes_per_launch")
        traffic_src = ("ncu --set full dram__bytes_read.sum + "
                       "dram__bytes_write.sum of the same kernel, from "
                       f"profiles/traffic_cfg3.json ({tj.get('source', '')})"
                       " -- not measured in this run")

    # ---- end to end through the public API from pinned host memory
    e2e = None
    if not args.no_e2e:
        if world == 1:
            xh = torch.from_numpy(x_np.astype(np.complex64)).pin_memory()
            hsig = ob.make_signal(xh, "complex", P, device="cpu")
            hout = torch.empty((NFIL, n_own), dtype=torch.complex64).pin_memory()
            pe = ob.plan(NS, M, "c2c", 0, NFFT)
            ob.convolve(hsig, fs, pe, out=hout)      # warm-up
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.e2e_steps):
                ob.convolve(hsig, fs, pe, out=hout)
            e1.record()
            e1.synchronize()
            e_ms = e0.elapsed_time(e1) / args.e2e_steps
            h2d = xh.numel() * 8
            path = ("make_signal(pinned host) + convolve(out=pinned host) "
                    "streaming row chunks (contiguous D2H)")
        else:
            # every rank: its owned samples from pinned host memory into its
            # halo'd buffer, halo exchange, its outputs in passes, each pass
            # copied to pinned host memory (sharding module's public API)
            own_h = torch.from_numpy(x_np.astype(np.complex64)).pin_memory()
            hout = torch.empty((NFIL, n_own), dtype=torch.complex64).pin_memory()
            tile_w = max(1, min(n_own, (256 << 20) // (8 * NFIL)))
            tile = torch.empty((NFIL, tile_w), dtype=torch.complex64, device=dev)

            def sink(g_a, g_b, t):
                hout[:, g_a - me.g_lo:g_b - me.g_lo].copy_(
                    t[:, :g_b - g_a], non_blocking=True)

            def e2e_step():
                hb.own.copy_(own_h, non_blocking=True)
                hb.exchange()
                convolve_shard_chunked(hb.buffer, me, p, fs.spectra_dev, NFIL,
                                       P, tile, sink)

            e2e_step()
            torch.cuda.synchronize()
            dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.e2e_steps):
                e2e_step()
            e1.record()
            e1.synchronize()
            e_ms = e0.elapsed_time(e1) / args.e2e_steps
            h2d = own_h.numel() * 8
            path = ("per rank: pinned shard -> HaloBuffer.own, NCCL halo "
                    "exchange, convolve_shard_chunked with a D2H sink per pass")
        te = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": outputs_per_step / (float(te.item()) * 1e-3),
               "unit": "samples/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(NFIL * n_own * 8),
               "ms_per_step": float(te.item()), "path": path}

    # ---- the paper's comparison point: cuFFT-based OLS (Algorithm 1,
    # convolve(variant="pipelined")) on the same shard, same N
    cufft = None
    if not args.no_cufft:
        pc = ob.plan(n_own, M, "c2c", 0, NFFT)
        sig_own = ob.make_signal(hb.own, "complex", P)
        fc = ob.transform_filters(ob.make_filterset(taps, 0, P, device=dev),
                                  pc, "natural")
        ob.convolve(sig_own, fc, pc, variant="pipelined", out=out)
        torch.cuda.synchronize()
        c_ms = []
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            ob.convolve(sig_own, fc, pc, variant="pipelined", out=out)
            e1.record()
            e1.synchronize()
            c_ms.append(e0.elapsed_time(e1))
        cm = statistics.median(c_ms)
        # the paper's comparison point in its fastest form here: per L2-sized
        # chunk, batched C2C over the overlapping windows (no gather),
        # multiply kernel, batched inverse, discard kernel
        ob.convolve(sig_own, fc, pc, variant="cufft_ols", out=out)
        torch.cuda.synchronize()
        k_ms = []
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            ob.convolve(sig_own, fc, pc, variant="cufft_ols", out=out)
            e1.record()
            e1.synchronize()
            k_ms.append(e0.elapsed_time(e1))
        km = statistics.median(k_ms)
        cufft = {"ms_per_step": km, "value": n_own * NFIL / (km * 1e-3) * world,
                 "unit": "samples/s", "speedup_fused": km / kmean,
                 "path": "convolve(variant='cufft_ols'), PAPER.md Algorithm "
                         "1 on L2-resident chunks: batched C2C over the "
                         "overlapping windows (idist = L), multiply kernel, "
                         "batched inverse C2C, discard kernel; same N (cuFFT "
                         "callbacks are not applied on this platform: "
                         "profiles/r02_cufft_callbacks.log)",
                 "eager": {"ms_per_step": cm, "speedup_fused": cm / kmean,
                           "path": "gather -> batched C2C cuFFT -> "
                                   "materialized multiply -> batched inverse "
                                   "C2C -> discard (chunked), same N"}}

    # the exact mode (the reference's arithmetic, bit-identical outputs) on the
    # same shard and grid, device-resident, one launch per step
    exact = None
    if world == 1 and not args.no_cufft:
        sig1 = ob.make_signal(hb.own, "complex", P)
        fs1 = ob.make_filterset(taps, 0, P, device=dev)
        ob.convolve(sig1, fs1, p, variant="fused_exact", out=out)
        torch.cuda.synchronize()
        x_ms = []
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            ob.convolve(sig1, fs1, p, variant="fused_exact", out=out)
            e1.record()
            e1.synchronize()
            x_ms.append(e0.elapsed_time(e1))
        xm = statistics.median(x_ms)
        exact = {"ms_per_step": xm, "value": n_own * NFIL / (xm * 1e-3),
                 "unit": "samples/s",
                 "path": "convolve(variant='fused_exact'): bit-identical to "
                         "the reference's fp32 fused_c2c (includes the exact "
                         "filter-spectra transform per call)"}

    # ---- BASELINE config 5 (the scaling shape), after the cfg3 buffers go
    cfg5 = None
    if not args.no_cfg5:
        del out, flush
        torch.cuda.empty_cache()
        cfg5 = run_cfg5(args, world, rank, dev, ob,
                        args.emulate_ranks if world == 1 else 0)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline()
        except Exception as exc:  # the oracle needs gcc-built oracle/build
            cpu = {"error": str(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "complex64 (fp32)",
            "data": "synthetic (reference generator convention, cli.py:41-55)",
            "config": {"workload": WORKLOAD, "signal_samples": ns_global,
                       "filters": NFIL, "taps": M, "fft_len": NFFT,
                       "parallelism": f"signal sharded over {world} GPU(s), "
                                      "persistent halo'd buffers, halo "
                                      "exchange by NCCL P2P",
                       "l2": "flushed between timed steps (256 MiB memset)"},
            "hbm_frac": achieved / hbm,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm,
                         "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_kind,
                         "alg_bytes_per_launch": alg_bytes,
                         "kernel_ms": kmean},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps,
            "cufft_ols": cufft,
            "exact_mode": exact,
            "cfg5": cfg5,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
