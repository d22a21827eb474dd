"""Device time of the fused engine in double precision on cfg2/cfg3 shapes."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import paper_1910_01972_b200 as ob  # noqa: E402
from cases import gen_inputs  # noqa: E402

for ns, m, nfil, n in [(1 << 22, 512, 32, 2048), (1 << 23, 400, 96, 2048),
                       (1 << 22, 64, 32, 256)]:
    x, taps = gen_inputs(ns, m, nfil)
    P = ob.Precision.double
    sig = ob.make_signal(x, "complex", P)
    p = ob.plan(ns, m, "c2c", 0, n)
    fs = ob.transform_filters(ob.make_filterset(taps, 0, P), p, "permuted")
    out = torch.empty((nfil, ns), dtype=torch.complex128, device="cuda")
    for _ in range(2):
        ob.convolve(sig, fs, p, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ob.convolve(sig, fs, p, out=out)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    t = float(np.median(ts))
    byts = 16 * ns * (1 + nfil)
    print(f"double ns={ns} m={m} F={nfil} N={n}: {t*1e3:.3f} ms "
          f"{ns * nfil / t:.3e} outputs/s {byts / t / 6.546e12 * 100:.1f}% HBM",
          flush=True)
