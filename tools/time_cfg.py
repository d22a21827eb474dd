"""Time the fused engine on BASELINE configs (CUDA events, device-resident).

    python tools/time_cfg.py cfg3 cfg2_n4096 ...   (OLSB_VARIANT selects policy)
Prints one line per config; also checks one golden case for parity.
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import paper_1910_01972_b200 as ob  # noqa: E402
from cases import CONV_GRID, conv_case_inputs, gen_inputs  # noqa: E402
from prof_cfg import CFG  # noqa: E402


def parity():
    c = np.load(os.path.join(ROOT, "tests/golden/conv_cases.npz"))
    worst = 0.0
    for i in (17, 18, 19, 20, 12):
        ns, m, nfil, n, origin, _ = CONV_GRID[i]
        x, taps = conv_case_inputs(i)
        P = ob.Precision.single
        y = ob.convolve(ob.make_signal(x, "complex", P),
                        ob.make_filterset(taps, origin, P),
                        ob.plan(ns, m, "c2c", origin, n)).cpu().numpy()
        ref = c[f"y_double_{i}"]
        e = np.max(np.linalg.norm(y - ref, axis=1) / np.linalg.norm(ref, axis=1))
        worst = max(worst, e)
    return worst


def time_cfg(name, reps=200):
    ns, m, nfil, n, *mode = CFG[name]
    mode = mode[0] if mode else "c2c"
    x, taps = gen_inputs(ns, m, nfil)
    P = ob.Precision.single
    if mode == "r2r":
        x, taps = x.real, taps.real
    sig = ob.make_signal(x, "real" if mode == "r2r" else "complex", P)
    p = ob.plan(ns, m, mode, 0, n)
    fs = ob.transform_filters(ob.make_filterset(taps, 0, P), p,
                              "natural" if mode == "r2r" else "permuted")
    out = torch.empty((nfil, ns), dtype=torch.float32 if mode == "r2r"
                      else torch.complex64, device="cuda")
    # back-to-back launches between two events (the host-side call overhead
    # overlaps the previous kernel; an event pair around each synchronous
    # call would count it for cells shorter than ~0.1 ms).  Windows of ~20 ms
    # with idle gaps: long sustained runs hit the 1000 W power cap and drop
    # the SM clock (tools/power_probe.py); median of 5 windows
    ex = ob.Executor(fs, p)
    xs = sig.samples
    for _ in range(3):
        ex(xs, out)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    ex(xs, out)
    e1.record()
    e1.synchronize()
    reps = max(3, min(reps, int(20.0 / max(e0.elapsed_time(e1), 1e-3))))
    ts = []
    for _ in range(5):
        time.sleep(0.25)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            ex(xs, out)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3 / reps)
    t = float(np.median(ts))
    byts = (4 if mode == "r2r" else 8) * ns * (1 + nfil)
    return t, byts / t / 6546.6e9


if __name__ == "__main__":
    v = os.environ.get("OLSB_VARIANT", "-")
    err = parity()
    for name in sys.argv[1:]:
        t, frac = time_cfg(name)
        ns, nfil = CFG[name][0], CFG[name][2]
        print(f"variant {v} {name}: {t*1e3:.3f} ms  {frac*100:.1f}% HBM  "
              f"{ns * nfil / t:.3e} outputs/s  parity {err:.2e}", flush=True)
