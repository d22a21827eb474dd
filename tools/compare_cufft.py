"""Fused engine vs the cuFFT-based OLS comparison point (north_star: >= 2x
at FFT lengths <= 4096).

    python tools/compare_cufft.py [cfg ...]

For every config: the fused engine at the config's N, and the cuFFT OLS
(`convolve(variant="pipelined")`: gather -> batched C2C (real path: R2C)
cuFFT -> multiply -> batched inverse C2C (C2R) -> discard, chunked over
segments, the paper's Algorithm 1) at the same N and at its own best N in {N, 8192, 16384}.  CUDA events,
median of 5 after 2 warm-ups, inputs resident, outputs preallocated.
Prints one JSON line per config.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import paper_1910_01972_b200 as ob  # noqa: E402
from cases import gen_inputs  # noqa: E402
from prof_cfg import CFG  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


def run(name):
    ns, m, nfil, n, *mode = CFG[name]
    mode = mode[0] if mode else "c2c"
    x, taps = gen_inputs(ns, m, nfil)
    if mode == "r2r":
        x, taps = x.real, taps.real
    P = ob.Precision.single
    sig = ob.make_signal(x, "real" if mode == "r2r" else "complex", P)
    fset = ob.make_filterset(taps, 0, P)
    out = torch.empty((nfil, ns), dtype=torch.float32 if mode == "r2r"
                      else torch.complex64, device="cuda")
    p = ob.plan(ns, m, mode, 0, n)
    fs = ob.transform_filters(fset, p,
                              "natural" if mode == "r2r" else "permuted")
    t_fused = timed(lambda: ob.convolve(sig, fs, p, out=out))
    ref = out.clone()
    res = {"cfg": name, "mode": mode, "n_s": ns, "m": m, "filters": nfil,
           "fft_len": n,
           "fused_ms": t_fused * 1e3,
           "fused_outputs_per_s": ns * nfil / t_fused}
    best = None
    for nc in sorted({n, 8192, 16384}):
        if nc < m:
            continue
        pc = ob.plan(ns, m, mode, 0, nc, max_fft_len=max(nc, 4096))
        fc = ob.transform_filters(fset, pc, "natural")
        t = timed(lambda: ob.convolve(sig, fc, pc, variant="pipelined",
                                      out=out), reps=3, warm=1)
        err = float((out - ref).abs().max() / ref.abs().max())
        res[f"cufft_ms_n{nc}"] = t * 1e3
        res[f"cufft_maxrel_vs_fused_n{nc}"] = err
        if best is None or t < best[1]:
            best = (nc, t)
        if nc == n:
            res["speedup_same_n"] = t / t_fused
    if mode == "c2c" and n <= 4096:
        # the L2-chunked cuFFT OLS (libolsb_cufft.so): no gather copy,
        # product chunks stay in L2
        fn = ob.transform_filters(fset, p, "natural")
        t = timed(lambda: ob.convolve(sig, fn, p, variant="cufft_ols",
                                      out=out), reps=5, warm=2)
        res["cufft_l2_ms"] = t * 1e3
        res["cufft_l2_maxrel_vs_fused"] = float(
            (out - ref).abs().max() / ref.abs().max())
        res["speedup_vs_cufft_l2"] = t / t_fused
    res["cufft_best_n"] = best[0]
    res["speedup_vs_cufft_best"] = best[1] / t_fused
    return res


if __name__ == "__main__":
    names = sys.argv[1:] or ["cfg1", "cfg2_n256", "cfg2_n512", "cfg2_n1024",
                             "cfg2_n2048", "cfg2_n4096", "cfg3", "cfg4_m8_f8",
                             "cfg4_m32_f8", "cfg3_r2r", "cfg2_n1024_r2r",
                             "cfg2_n4096_r2r"]
    for nm in names:
        print(json.dumps(run(nm)), flush=True)
