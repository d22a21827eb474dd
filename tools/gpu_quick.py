"""Quick GPU sanity + timing probe (development tool, not a test)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import paper_1910_01972_b200 as ob  # noqa: E402
from cases import CONV_GRID, conv_case_inputs, gen_inputs  # noqa: E402

P = ob.Precision


def rel_l2(got, ref):
    got = np.asarray(got)
    ref = np.asarray(ref)
    num = np.sqrt(np.sum(np.abs(got - ref) ** 2, axis=-1))
    den = np.sqrt(np.sum(np.abs(ref) ** 2, axis=-1))
    return float(np.max(num / np.maximum(den, 1e-300)))


def main():
    c = np.load(os.path.join(ROOT, "tests/golden/conv_cases.npz"))
    worst = {"single": 0.0, "double": 0.0}
    for i, (ns, m, nfil, n, origin, rt) in enumerate(CONV_GRID):
        x, taps = conv_case_inputs(i)
        for prec in (P.single, P.double):
            sig = ob.make_signal(x, "complex", prec)
            fs = ob.make_filterset(taps, origin, prec)
            p = ob.plan(ns, m, "c2c", origin, n)
            y = ob.convolve(sig, fs, p).cpu().numpy()
            e = rel_l2(y, c[f"y_double_{i}"])
            worst[prec.value] = max(worst[prec.value], e)
            if not np.all(np.isfinite(y)) or e > (1e-5 if prec is P.single else 1e-11):
                print("BAD", i, prec.value, e, flush=True)
    print("worst rel L2", worst, flush=True)

    for name, ns, m, nfil, n in [("cfg1", 1 << 20, 64, 1, 1024),
                                 ("cfg3", 1 << 23, 400, 96, 2048),
                                 ("cfg2_n4096", 1 << 22, 1024, 32, 4096),
                                 ("cfg2_n256", 1 << 22, 64, 32, 256),
                                 ("cfg4_m8_f8", 1 << 24, 8, 8, 64)]:
        x, taps = gen_inputs(ns, m, nfil)
        sig = ob.make_signal(x, "complex", P.single)
        fs = ob.make_filterset(taps, 0, P.single)
        p = ob.plan(ns, m, "c2c", 0, n)
        fs = ob.transform_filters(fs, p, "permuted")
        out = torch.empty((nfil, ns), dtype=torch.complex64, device="cuda")
        for _ in range(3):
            ob.convolve(sig, fs, p, out=out)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            ob.convolve(sig, fs, p, out=out)
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1) / reps * 1e-3
        byts = 8 * ns * (1 + nfil)
        print(f"{name}: {t*1e3:.3f} ms  {ns*nfil/t:.3e} out/s  "
              f"{byts/t/1e9:.0f} GB/s ({byts/t/6546.6e9*100:.1f}% of 6546.6)",
              flush=True)


if __name__ == "__main__":
    main()
