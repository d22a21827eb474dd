"""Kernel time of variant="fused_exact" (the reference's arithmetic) against
the default fused engine on cfg3 and a cfg2 cell (CUDA events, back-to-back
launches, median of 5 windows)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden")]
import paper_1910_01972_b200 as ob  # noqa: E402
from cases import gen_inputs  # noqa: E402

for ns, m, nfil, n in [(1 << 23, 400, 96, 2048), (1 << 22, 256, 32, 1024)]:
    x, taps = gen_inputs(ns, m, nfil)
    P = ob.Precision.single
    sig = ob.make_signal(x, "complex", P)
    p = ob.plan(ns, m, "c2c", 0, n)
    fs = ob.transform_filters(ob.make_filterset(taps, 0, P), p, "permuted")
    out = torch.empty((nfil, ns), dtype=torch.complex64, device="cuda")
    res = {}
    for v in ("fused", "fused_exact"):
        for _ in range(2):
            ob.convolve(sig, fs, p, variant=v, out=out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                ob.convolve(sig, fs, p, variant=v, out=out)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) / 5)
        res[v] = float(np.median(ts))
    byts = 8 * ns * (1 + nfil)
    print(f"ns={ns} M={m} F={nfil} N={n}: fused {res['fused']:.3f} ms, "
          f"fused_exact {res['fused_exact']:.3f} ms "
          f"({byts / res['fused_exact'] / 1e-3 / 6546.6e9 * 100:.1f}% HBM)",
          flush=True)
