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

# round 2: range / host-streaming / shard entries with every post-process,
# the M = 1 derivative, and the cuFFT-OLS comparison point
from paper_1910_01972_b200.ols import fused_range_launch, _engine_spectra  # noqa: E402
from paper_1910_01972_b200.sharding import convolve_shard, make_shards  # noqa: E402
for n, m in ((256, 1), (1024, 65), (2048, 400), (4096, 512)):
    ns = 5 * n + 33
    for mode in ("c2c", "r2r"):
        real = mode == "r2r"
        x = rng.standard_normal(ns) if real else (rng.standard_normal(ns)
                                                  + 1j * rng.standard_normal(ns))
        taps = rng.standard_normal((3, m)) if real else (
            rng.standard_normal((3, m)) + 1j * rng.standard_normal((3, m)))
        p = ob.plan(ns, m, mode, m // 2, n)
        vk = "real" if real else "complex"
        fs = ob.transform_filters(ob.make_filterset(taps, m // 2, P), p,
                                  "natural" if real else "permuted")
        sig = ob.make_signal(x, vk, P)
        for ppk in ("none", "scale", "magnitude_squared", "derivative"):
            if ppk == "magnitude_squared" and not real:
                continue
            pp = ob.PostProcSpec(ppk, 0.5) if ppk == "scale" else ob.PostProcSpec(ppk)
            dev = ob.convolve(sig, fs, p, postproc=pp)
            host = torch.empty(tuple(dev.shape), dtype=dev.dtype).pin_memory()
            hsig = ob.make_signal(sig.samples.cpu().pin_memory(), vk, P, device="cpu")
            ob.convolve(hsig, fs, p, postproc=pp, out=host, chunk_segments=3)
            torch.cuda.synchronize()
            assert torch.equal(host, dev.cpu()), (n, m, mode, ppk)
            for sh in make_shards(p, 3, postproc=pp):
                if sh.g_hi > sh.g_lo:
                    xl = sig.samples[sh.x_lo:sh.x_hi].clone()
                    got = convolve_shard(xl, sh, p, fs, postproc=pp)
                    torch.cuda.synchronize()
                    assert torch.equal(got, dev[:, sh.g_lo:sh.g_hi]), (n, mode, ppk)
        if not real:
            y = ob.convolve(sig, ob.make_filterset(taps, m // 2, P), p,
                            variant="cufft_ols")
            torch.cuda.synchronize()
            assert torch.isfinite(y).all()
print("sanitize cells done")
