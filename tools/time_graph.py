"""Kernel-bound timing of small cells: CUDA-graph replay of 20 back-to-back
Executor launches (no host overhead), median of 5 replays.

    python tools/time_graph.py cfg1 [cfg4_m8_f1 ...]   (OLSB_VARIANT selects policy)
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden"),
                os.path.join(ROOT, "tools")]
import paper_1910_01972_b200 as ob  # noqa: E402
from cases import gen_inputs  # noqa: E402
from prof_cfg import CFG  # noqa: E402

try:
    import json
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        PEAK = float(json.load(f)["hbm_gbs"]) * 1e9
except Exception:
    PEAK = 6650e9

for name in sys.argv[1:]:
    ns, m, nfil, n, *_ = CFG[name]
    x, taps = gen_inputs(ns, m, nfil)
    P = ob.Precision.single
    sig = ob.make_signal(x, "complex", P)
    p = ob.plan(ns, m, "c2c", 0, n)
    fs = ob.transform_filters(ob.make_filterset(taps, 0, P), p, "permuted")
    out = torch.empty((nfil, ns), dtype=torch.complex64, device="cuda")
    ex = ob.Executor(fs, p)
    run = ex.graph(sig.samples, out, launches=20)
    ts = []
    for _ in range(6):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 20)
    t = float(np.median(ts[1:]))
    byts = 8 * ns * (1 + nfil)
    print(f"variant {os.environ.get('OLSB_VARIANT', '-')} {name}: {t * 1e3:.1f} us "
          f"{byts / (t * 1e-3) / PEAK * 100:.1f}% HBM", flush=True)
