"""Pin the CPU oracle (oracle/) against the reference's own outputs.

The fixtures in tests/golden were produced by running the reference package
itself (tests/golden/make_golden.py).  The oracle restates the reference's
loops in C with the same IEEE operation order, so single AND double precision
agree bit for bit; these tests fail on any drift.
"""

import numpy as np
import pytest

import oracle
from cases import CONV_GRID, PP_GRID, conv_case_inputs, pp_case_inputs, pp_scale
from conftest import rel_err


def _bitrev_perm(n):
    bits = n.bit_length() - 1
    out = []
    for k in range(n):
        r, i = 0, k
        for _ in range(bits):
            r = (r << 1) | (i & 1)
            i >>= 1
        out.append(r)
    return np.array(out)


@pytest.mark.parametrize("precision", ["single", "double"])
def test_fft_bit_exact_vs_reference(golden, precision):
    g = golden["fft"]
    n = 4
    while n <= 4096:
        x = g[f"x_{n}"].astype(oracle._cdtype(precision))
        assert np.array_equal(oracle.fft_forward_permuted(x, precision),
                              g[f"fwd_{precision}_{n}"]), n
        assert np.array_equal(oracle.fft_inverse_permuted(x, precision),
                              g[f"inv_{precision}_{n}"]), n
        n *= 2


def test_fft_known_answers():
    # test_fft.py:103-122 of the reference
    out = oracle.fft_forward_permuted([0, 1, 2, 3], "double")
    assert np.allclose(out, [6, -2, -2 + 2j, -2 - 2j])
    assert np.allclose(oracle.fft_forward_permuted([1, 0, 0, 0], "double"),
                       np.ones(4))
    assert np.allclose(oracle.fft_forward_permuted([1, 1, 1, 1], "double"),
                       [4, 0, 0, 0])
    assert np.allclose(oracle.fft_inverse_permuted([6, -2, -2 + 2j, -2 - 2j],
                                                   "double"), [0, 1, 2, 3])
    assert np.allclose(oracle.fft_inverse_permuted([4, 0, 0, 0], "double"),
                       np.ones(4))


def test_transform_filters_known_answer():
    # test_ols.py:91-98: [1,1] at N=4 -> permuted [2, 0, 1-i, 1+i]
    spec = oracle.transform_filters([[1 + 0j, 1 + 0j]], 4, "double")
    assert np.allclose(spec[0], [2, 0, 1 - 1j, 1 + 1j])
    delta = oracle.transform_filters([[1 + 0j]], 8, "double")
    assert np.allclose(delta[0], np.ones(8))


@pytest.mark.parametrize("precision", ["single", "double"])
def test_spectra_bit_exact_vs_reference(golden, precision):
    g = golden["spectra"]
    for key in g.files:
        if not key.startswith("taps_"):
            continue
        _, n, m = key.split("_")
        spec = oracle.transform_filters(g[key].astype(oracle._cdtype(precision)),
                                        int(n), precision)
        assert np.array_equal(spec, g[f"spec_{precision}_{n}_{m}"]), key


@pytest.mark.parametrize("case", range(len(CONV_GRID)))
def test_fused_bit_exact_vs_reference(golden, case):
    ns, m, nfil, n, origin, _ = CONV_GRID[case]
    x, taps = conv_case_inputs(case)
    g = golden["conv"]
    for precision in ("single", "double"):
        dt = oracle._cdtype(precision)
        y = oracle.fused_convolve(x.astype(dt), taps.astype(dt), n, origin,
                                  precision, threads=3)
        assert np.array_equal(y, g[f"y_{precision}_{case}"]), precision
    if f"direct_{case}" in g.files:
        d = oracle.direct_convolve(x, taps, origin, threads=2)
        assert rel_err(d, g[f"direct_{case}"]) < 1e-13


def test_fused_split_invariance():
    # any split of the segment range gives identical bits (ols.py:20-23)
    x, taps = conv_case_inputs(12)
    ns, m, nfil, n, origin, _ = CONV_GRID[12]
    a = oracle.fused_convolve(x, taps, n, origin, "single", threads=1)
    b = oracle.fused_convolve(x, taps, n, origin, "single", threads=5)
    assert np.array_equal(a, b)


def test_direct_window_matches_full():
    x, taps = conv_case_inputs(10)
    ns, m, nfil, n, origin, _ = CONV_GRID[10]
    full = oracle.direct_convolve(x, taps, origin)
    for a, b in ((0, 300), (1000, 1500), (ns - 200, ns)):
        w = oracle.direct_window(x, taps, origin, a, b)
        assert rel_err(w, full[:, a:b]) < 1e-13


def test_cfg_golden_windows_consistent(golden):
    # the oracle at full cfg1 size reproduces the reference's fp64 windows
    from cases import gen_inputs
    g = golden["cfg"]
    ns, m, nfil, n = (int(v) for v in g["cfg1_params"])
    x, taps = gen_inputs(ns, m, nfil)
    y = oracle.fused_convolve(x, taps, n, 0, "double")
    starts = g["cfg1_starts"]
    win = np.stack([y[:, s:s + 256] for s in starts], axis=1)
    assert rel_err(win, g["cfg1_win"]) < 1e-6   # fixture stored as complex64
    assert np.allclose(np.sum(np.abs(y) ** 2, axis=1), g["cfg1_sumsq"],
                       rtol=1e-12)


@pytest.mark.parametrize("case", range(len(PP_GRID)))
def test_pp_fixtures_match_direct_oracle(golden, case):
    """The reference's real path / magnitude_squared outputs (pp_cases.npz)
    agree with the oracle's float64 direct convolution (pins the fixtures the
    GPU r2r / abs2 parity tests use)."""
    ns, m, nfil, n, origin, mode, ppk = PP_GRID[case]
    x, taps = pp_case_inputs(case)
    y = oracle.direct_convolve(x, taps, origin)
    if ppk == "scale":
        y = y * pp_scale(case)
    if mode == "r2r":
        y = y.real
        if ppk == "magnitude_squared":
            y = y * y
    elif ppk == "magnitude_squared":
        y = np.abs(y) ** 2
    if ppk == "derivative":   # postproc.py:44-85, both ends one-sided
        d = np.empty_like(y)
        if ns == 1:
            d[:] = 0
        else:
            d[:, 1:-1] = 0.5 * (y[:, 2:] - y[:, :-2])
            d[:, 0] = y[:, 1] - y[:, 0]
            d[:, -1] = y[:, -1] - y[:, -2]
        y = d
    ref = golden["pp"][f"y_double_{case}"]
    assert ref.shape == (nfil, ns)
    assert np.isrealobj(ref) == (mode == "r2r" or ppk == "magnitude_squared")
    assert rel_err(ref, y) < 1e-10


@pytest.mark.parametrize("case", [i for i, c in enumerate(PP_GRID)
                                  if c[5] == "c2c" and c[6] == "scale"])
def test_fused_scale_bit_exact_vs_reference(golden, case):
    """postproc scale with a factor fp32 cannot represent (0.3): the
    reference rounds float64(pp_c) x sample once into complex64 (_store kind
    1, _kernels_nb.py:223-225); the oracle reproduces its fp32 output bit for
    bit (the GPU exact mode is checked against the same fixtures)."""
    ns, m, nfil, n, origin, mode, ppk = PP_GRID[case]
    x, taps = pp_case_inputs(case)
    y = oracle.fused_convolve(x, taps, n, origin, "single", pp_kind=1,
                              pp_c=pp_scale(case))
    assert np.array_equal(y, golden["pp"][f"y_single_{case}"])
