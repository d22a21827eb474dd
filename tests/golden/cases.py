"""Deterministic case definitions shared by the golden generator and the tests.

Inputs are never stored in the fixtures: they are regenerated from numpy's
PCG64 seeded streams, which are bit-reproducible on every platform.  The bench
generator follows the reference's own convention (cli.py:41-55).
"""

from __future__ import annotations

import numpy as np


def gen_inputs(ns, m, nfil, origin=0, seed=0):
    """The reference bench generator, cli.py:41-55 (c2c tag = 0): complex
    N(0,1) + i N(0,1) signal and taps, drawn in that order."""
    rng = np.random.default_rng([seed, ns, m, nfil, origin, 0])
    x = rng.standard_normal(ns) + 1j * rng.standard_normal(ns)
    taps = rng.standard_normal((nfil, m)) + 1j * rng.standard_normal((nfil, m))
    return x, taps


# (n_s, m, nfil, n, origin, real_taps)
CONV_GRID = [
    (1, 5, 2, 64, 2, False),          # single sample  (test_ols.py:254-263)
    (63, 5, 2, 64, 2, False),
    (64, 5, 2, 64, 0, False),
    (65, 5, 2, 64, 4, False),
    (1000, 1, 1, 4, 0, False),        # M = 1, nothing discarded
    (1000, 1, 3, 64, 0, False),
    (1000, 4, 2, 4, 3, False),        # M = N  -> L = 1
    (777, 64, 1, 64, 0, False),       # M = N
    (5000, 3, 2, 64, 1, False),       # test_ols.py:138-150 grid
    (5000, 33, 2, 128, 16, False),
    (5000, 257, 2, 1024, 128, False),
    (4096, 57, 2, 256, 0, False),     # segment-size invariance cell
    (10000, 33, 2, 256, 0, False),    # workers bit-identical cell
    (6000, 65, 3, 512, 32, False),    # variant-equivalence cell
    (3000, 17, 4, 32, 0, True),       # real taps on a complex signal
    (3000, 9, 2, 16, 8, False),
    (2000, 7, 2, 8, 3, False),
    (9000, 129, 2, 2048, 64, False),
    (9000, 400, 3, 2048, 0, False),   # FDAS shape, small
    (12000, 1025, 1, 4096, 512, False),
    (9000, 2049, 1, 4096, 0, False),
    (9000, 250, 2, 256, 249, False),  # origin = M-1
]


def conv_case_inputs(i):
    ns, m, nfil, n, origin, real_taps = CONV_GRID[i]
    rng = np.random.default_rng([30, i, ns, m, nfil, n, origin])
    x = rng.standard_normal(ns) + 1j * rng.standard_normal(ns)
    if real_taps:
        taps = rng.standard_normal((nfil, m))
    else:
        taps = rng.standard_normal((nfil, m)) + 1j * rng.standard_normal((nfil, m))
    return x, taps


# real path + post-processing cells:
# (n_s, m, nfil, n, origin, mode, postproc)
PP_GRID = [
    (1, 5, 2, 64, 2, "r2r", "none"),          # single sample
    (63, 5, 2, 64, 2, "r2r", "none"),
    (65, 5, 2, 64, 4, "r2r", "scale"),
    (1000, 1, 3, 8, 0, "r2r", "none"),        # M = 1, N = 8 (r2r floor)
    (777, 64, 1, 64, 0, "r2r", "none"),       # M = N
    (5000, 33, 2, 128, 16, "r2r", "none"),
    (5000, 257, 2, 1024, 128, "r2r", "magnitude_squared"),
    (9000, 400, 3, 2048, 0, "r2r", "none"),   # FDAS shape, small
    (9000, 129, 2, 2048, 64, "r2r", "scale"),
    (12000, 1025, 1, 4096, 512, "r2r", "none"),
    (10000, 33, 2, 256, 0, "r2r", "none"),
    (6000, 65, 3, 512, 32, "c2c", "magnitude_squared"),
    (9000, 400, 2, 2048, 0, "c2c", "magnitude_squared"),
    (3000, 9, 2, 16, 8, "c2c", "magnitude_squared"),
    # derivative: halo geometry (l_eff = L - 2), one-sided at the signal ends
    (5000, 33, 2, 128, 16, "c2c", "derivative"),
    (9000, 400, 2, 2048, 0, "c2c", "derivative"),
    (12000, 1025, 1, 4096, 512, "c2c", "derivative"),
    (65, 5, 2, 64, 4, "c2c", "derivative"),
    (2, 3, 1, 8, 1, "c2c", "derivative"),
    (1000, 1, 2, 64, 0, "c2c", "derivative"),    # M = 1: seam recompute
    (9000, 400, 3, 2048, 0, "r2r", "derivative"),
    (5000, 33, 2, 128, 16, "r2r", "derivative"),
    (1000, 1, 2, 8, 0, "r2r", "derivative"),
    # complex scale with a factor fp32 cannot represent: the reference
    # multiplies in float64 and rounds once (_store kind 1)
    (6000, 65, 3, 512, 32, "c2c", "scale"),
    (9000, 400, 2, 2048, 0, "c2c", "scale"),
]


def pp_case_inputs(i):
    ns, m, nfil, n, origin, mode, pp = PP_GRID[i]
    rng = np.random.default_rng([40, i, ns, m, nfil, n, origin])
    if mode == "r2r":
        return rng.standard_normal(ns), rng.standard_normal((nfil, m))
    x = rng.standard_normal(ns) + 1j * rng.standard_normal(ns)
    taps = rng.standard_normal((nfil, m)) + 1j * rng.standard_normal((nfil, m))
    return x, taps


PP_SCALE = 0.75          # r2r scale cells
PP_SCALE_C2C = 0.3       # c2c scale cells (not representable in fp32)


def pp_scale(i):
    """postproc scale factor of PP_GRID cell i (1.0 unless it is a scale cell)."""
    mode, ppk = PP_GRID[i][5], PP_GRID[i][6]
    if ppk != "scale":
        return 1.0
    return PP_SCALE if mode == "r2r" else PP_SCALE_C2C

# BASELINE.json configs 1-4 (SURVEY §8 geometry table); cfg5 (2^30) cannot
# run on the reference and is checked by windows against the oracle instead.
CFGS = [
    ("cfg1", 1 << 20, 64, 1, 1024),
    ("cfg2_n256", 1 << 22, 64, 32, 256),
    ("cfg2_n512", 1 << 22, 128, 32, 512),
    ("cfg2_n1024", 1 << 22, 256, 32, 1024),
    ("cfg2_n2048", 1 << 22, 512, 32, 2048),
    ("cfg2_n4096", 1 << 22, 1024, 32, 4096),
    ("cfg3", 1 << 23, 400, 96, 2048),
    ("cfg4_m8_f1", 1 << 24, 8, 1, 64),
    ("cfg4_m16_f8", 1 << 24, 16, 8, 64),
    ("cfg4_m32_f8", 1 << 24, 32, 8, 128),
]
N_WIN = 8
WIN = 256


def window_starts(ns, l):
    """Fixed probe windows: both signal ends, segment seams, interior."""
    cands = [0, l - WIN // 2, 3 * l - 7, ns // 3, ns // 2 + 11,
             (2 * ns) // 3, ns - WIN - 5 * l, ns - WIN]
    return np.array([min(max(c, 0), ns - WIN) for c in cands[:N_WIN]],
                    dtype=np.int64)
