"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
itself (``olsconv`` from /root/reference/pkg/src, numba backend).

This script is the only thing in the repo that imports the reference; it runs
in the build container (the reference does not exist on the GPU box) and its
outputs are committed as small .npz files.  Run:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Fixtures
--------
fft_permuted.npz   forward/inverse reorder-free transforms (fft.py:112-125,
                   _kernels_nb.py:11-51) for N = 4..4096, both precisions.
spectra.npz        transform_filters(..., "permuted") (ols.py:168-205).
conv_cases.npz     convolve(variant="fused") c2c (ols.py:257-360) on a grid of
                   small cells incl. every edge case of SURVEY §8(a): first /
                   last segment, M=1, M=N, N_s < L, origin > 0, real taps.
pp_cases.npz       the real (r2r) path and the magnitude_squared epilogue
                   (fused_r2r / fused_c2c_abs2) on a grid of small cells.
io/                OLS1 binary / text sample files written by the reference's
                   io.write_samples (CLI file-format compatibility).
cfg_windows.npz    BASELINE.json configs 1-4 at FULL size: float64 reference
                   output on fixed windows + per-filter checksums.  Inputs are
                   regenerated anywhere from the reference's own generator
                   convention (cli.py:41-55), so only outputs are stored.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import olsconv as oc  # noqa: E402  (the reference)

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from cases import (CFGS, CONV_GRID, PP_GRID, WIN, pp_scale,  # noqa: E402
                   conv_case_inputs, gen_inputs, pp_case_inputs,
                   window_starts)
from olsconv import Precision  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
WORKERS = os.cpu_count() or 1


def fft_fixtures():
    out = {}
    n = 4
    while n <= 4096:
        rng = np.random.default_rng([10, n])
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        out[f"x_{n}"] = x
        for prec in Precision:
            p = oc.make_plan(n, "ct_dif_permuted", prec)
            xin = x.astype(prec.complex_dtype)
            fwd = oc.fft_forward_permuted(xin, p)
            inv = oc.fft_inverse_permuted(xin, p)
            out[f"fwd_{prec.value}_{n}"] = fwd
            out[f"inv_{prec.value}_{n}"] = inv
        n *= 2
    np.savez_compressed(os.path.join(HERE, "fft_permuted.npz"), **out)


def spectra_fixtures():
    out = {}
    cases = [(4, 2), (8, 1), (16, 5), (32, 32), (64, 33), (128, 64),
             (256, 100), (512, 129), (1024, 257), (2048, 400), (4096, 1025)]
    for n, m in cases:
        rng = np.random.default_rng([20, n, m])
        taps = rng.standard_normal((3, m)) + 1j * rng.standard_normal((3, m))
        out[f"taps_{n}_{m}"] = taps
        for prec in Precision:
            fs = oc.make_filterset(taps, 0, prec)
            p = oc.plan(1000, m, "c2c", 0, n)
            cached = oc.transform_filters(fs, p, "permuted")
            out[f"spec_{prec.value}_{n}_{m}"] = np.array(cached.spectra)
    np.savez_compressed(os.path.join(HERE, "spectra.npz"), **out)


def conv_fixtures():
    out = {"grid": np.array([[c[0], c[1], c[2], c[3], c[4], int(c[5])]
                             for c in CONV_GRID], dtype=np.int64)}
    for i, (ns, m, nfil, n, origin, real_taps) in enumerate(CONV_GRID):
        x, taps = conv_case_inputs(i)
        p = oc.plan(ns, m, "c2c", origin, n)
        for prec in Precision:
            sig = oc.make_signal(x, "complex", prec)
            fs = oc.make_filterset(taps, origin, prec)
            y = oc.convolve(sig, fs, p, variant="fused", workers=1)
            assert np.all(np.isfinite(y))
            out[f"y_{prec.value}_{i}"] = y
        if ns * m * nfil <= 2_000_000:
            sig = oc.make_signal(x, "complex", Precision.double)
            fs = oc.make_filterset(taps, origin, Precision.double)
            out[f"direct_{i}"] = oc.direct_convolve(sig, fs).outputs
    np.savez_compressed(os.path.join(HERE, "conv_cases.npz"), **out)


def pp_fixtures():
    """Real path (fused_r2r, _kernels_nb.py:312-337) and magnitude_squared
    (fused_c2c_abs2, :288-309) through the reference's convolve."""
    out = {}
    for i, (ns, m, nfil, n, origin, mode, ppk) in enumerate(PP_GRID):
        x, taps = pp_case_inputs(i)
        p = oc.plan(ns, m, mode, origin, n)
        pp = oc.PostProcSpec(ppk, pp_scale(i))
        vk = "real" if mode == "r2r" else "complex"
        for prec in Precision:
            sig = oc.make_signal(x, vk, prec)
            fs = oc.make_filterset(taps, origin, prec)
            y = oc.convolve(sig, fs, p, variant="fused", postproc=pp,
                            workers=1)
            assert np.all(np.isfinite(y))
            out[f"y_{prec.value}_{i}"] = y
    np.savez_compressed(os.path.join(HERE, "pp_cases.npz"), **out)


def io_fixtures():
    """OLS1 binary and text sample files written by the reference's own
    writer (io.py), for byte-level compatibility tests."""
    from olsconv.io import write_samples
    d = os.path.join(HERE, "io")
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng([90])
    arrays = {
        "real_single": rng.standard_normal(37).astype(np.float32),
        "real_double": rng.standard_normal(5),
        "complex_single": (rng.standard_normal(11)
                           + 1j * rng.standard_normal(11)).astype(np.complex64),
        "complex_double": rng.standard_normal(4) + 1j * rng.standard_normal(4),
    }
    for name, arr in arrays.items():
        write_samples(os.path.join(d, f"{name}.bin"), arr)
        write_samples(os.path.join(d, f"{name}.txt"), arr)
    np.savez_compressed(os.path.join(d, "arrays.npz"), **arrays)


def cfg_fixtures():
    out = {}
    for name, ns, m, nfil, n in CFGS:
        tic = time.time()
        x, taps = gen_inputs(ns, m, nfil)
        p = oc.plan(ns, m, "c2c", 0, n)
        sig = oc.make_signal(x, "complex", Precision.double)
        fs = oc.make_filterset(taps, 0, Precision.double)
        y = oc.convolve(sig, fs, p, variant="fused", workers=WORKERS)
        starts = window_starts(ns, p.valid_len)
        win = np.stack([y[:, s:s + WIN] for s in starts], axis=1)
        out[f"{name}_params"] = np.array([ns, m, nfil, n], dtype=np.int64)
        out[f"{name}_starts"] = starts
        out[f"{name}_win"] = win.astype(np.complex64)
        out[f"{name}_sumsq"] = np.sum(np.abs(y) ** 2, axis=1)
        out[f"{name}_sum"] = np.sum(y, axis=1)
        print(f"{name}: {time.time() - tic:.1f}s", flush=True)
        del y, sig, x
    np.savez_compressed(os.path.join(HERE, "cfg_windows.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["fft", "spectra", "conv", "pp", "io", "cfg"]
    if "fft" in which:
        fft_fixtures()
    if "spectra" in which:
        spectra_fixtures()
    if "conv" in which:
        conv_fixtures()
    if "pp" in which:
        pp_fixtures()
    if "io" in which:
        io_fixtures()
    if "cfg" in which:
        cfg_fixtures()
    print("backend:", oc.backend_name())
