"""Small cells of every FFT length and mode, for compute-sanitizer runs.

    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_cells.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1910_01972_b200 as ob  # noqa: E402

P = ob.Precision.single
rng = np.random.default_rng(5)
for n in (8, 16, 64, 256, 512, 1024, 2048, 4096):
    m = max(1, n // 4)
    ns = 3 * n + 17
    for mode, ppk in (("c2c", "none"), ("c2c", "derivative"),
                      ("c2c", "magnitude_squared"), ("r2r", "none")):
        real = mode == "r2r"
        x = rng.standard_normal(ns) if real else (rng.standard_normal(ns)
                                                  + 1j * rng.standard_normal(ns))
        taps = rng.standard_normal((2, m)) if real else (
            rng.standard_normal((2, m)) + 1j * rng.standard_normal((2, m)))
        p = ob.plan(ns, m, mode, 0, n)
        y = ob.convolve(ob.make_signal(x, "real" if real else "complex", P),
                        ob.make_filterset(taps, 0, P), p,
                        postproc=ob.PostProcSpec(ppk))
        torch.cuda.synchronize()
        assert torch.isfinite(y).all(), (n, mode, ppk)
        if mode == "c2c" and ppk in ("none", "magnitude_squared"):
            y = ob.convolve(ob.make_signal(x, "complex", P),
                            ob.make_filterset(taps, 0, P), p,
                            postproc=ob.PostProcSpec(ppk), variant="fused_exact")
            torch.cuda.synchronize()
            assert torch.isfinite(y).all(), (n, "exact", ppk)
print("sanitize cells done")
