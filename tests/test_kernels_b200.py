"""The reference-side kernel backend (paper_1910_01972_b200.kernels_b200):
the reference's ``K.*`` numpy contract (``_kernels_nb.py``) served by the
engine, as ``backend.py:18-36`` would load it.

CPU: the module exports the reference's hot-path names with its argument
lists.  GPU: called exactly as the reference's ``convolve`` calls ``K`` --
its own permuted spectra (``tests/golden/spectra.npz``, made by the
reference), uneven ``[seg_lo, seg_hi)`` worker ranges into a NaN-prefilled
``out`` -- every call writes only its windows; the exact mode is bit-identical
to the reference's fp32 kernels (the pinned oracle), the fast mode within the
fp32 tolerance of the float64 direct convolution.
"""

import inspect

import numpy as np
import pytest

import oracle
from conftest import has_gpu, rel_l2_per_filter

# argument lists of the reference's kernels (_kernels_nb.py:54-63, 265-337)
REF_SIGNATURES = {
    "dif_fwd_batch": ["mat", "tw"],
    "dit_inv_batch": ["mat", "twc"],
    "fused_c2c": ["x", "spectra", "tw", "twc", "m", "origin", "l_eff", "t0",
                  "win_off", "seg_lo", "seg_hi", "pp_kind", "pp_c", "h0",
                  "out", "buf", "spec_buf"],
    "fused_c2c_abs2": ["x", "spectra", "tw", "twc", "m", "origin", "l_eff",
                       "t0", "win_off", "seg_lo", "seg_hi", "h0", "out", "buf",
                       "spec_buf"],
    "fused_r2r": ["x", "spectra", "tw_half", "tw_half_conj", "pack_tw",
                  "pack_tw_conj", "m", "origin", "l_eff", "t0", "win_off",
                  "seg_lo", "seg_hi", "pp_kind", "pp_c", "h0", "out", "rbuf",
                  "z_scr", "bins", "prod"],
}


def test_exports_reference_kernel_signatures():
    from paper_1910_01972_b200 import kernels_b200 as K
    for name, args in REF_SIGNATURES.items():
        assert list(inspect.signature(getattr(K, name)).parameters) == args, name


def _splits(n_seg):
    """uneven worker ranges like _chunk_bounds with a remainder"""
    a = max(1, n_seg // 3)
    b = min(n_seg, a + max(1, n_seg // 5))
    return [(0, a), (a, b), (b, n_seg)]


CASES = [(64, 33, 3000, 5), (512, 129, 20000, 17), (2048, 400, 30000, 0),
         (4096, 1025, 20000, 512)]


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,ns,origin", CASES)
def test_fused_c2c_reference_contract(golden, n, m, ns, origin):
    assert has_gpu()
    from paper_1910_01972_b200 import kernels_b200 as K
    spectra = golden["spectra"][f"spec_single_{n}_{m}"]
    taps = golden["spectra"][f"taps_{n}_{m}"]
    spectra = np.array(spectra, dtype=np.complex64)
    spectra.flags.writeable = False          # a cached FilterSet's spectra
    rng = np.random.default_rng([95, n, ns])
    x = (rng.standard_normal(ns) + 1j * rng.standard_normal(ns)).astype(np.complex64)
    tw, twc = oracle.tables(n, "single")
    l_eff, t0, win_off = oracle.geometry(m, origin, n)
    n_seg = -(-ns // l_eff)
    h0 = taps[:, 0].astype(np.complex64)
    want_exact = oracle.fused_convolve(x, taps, n, origin, "single")
    ref64 = oracle.direct_convolve(x, taps, origin)
    for exact in (True, False):
        K.EXACT = exact
        try:
            out = np.full((taps.shape[0], ns), np.nan, np.complex64)
            for lo, hi in _splits(n_seg):
                K.fused_c2c(x, spectra, tw, twc, m, origin, l_eff, t0, win_off,
                            lo, hi, 0, 1.0, h0, out, None, None)
                g_hi = min(hi * l_eff, ns)
                assert np.all(np.isfinite(out[:, :g_hi]))     # its windows
                assert np.all(np.isnan(out[:, g_hi:]))        # nothing else
        finally:
            K.EXACT = True
        if exact:
            assert np.array_equal(out, want_exact)
        else:
            assert rel_l2_per_filter(out, ref64) <= 1e-5


@pytest.mark.gpu
def test_fused_c2c_scale_abs2_and_transforms(golden):
    assert has_gpu()
    from paper_1910_01972_b200 import kernels_b200 as K
    n, m, ns, origin = 512, 129, 12000, 3
    spectra = np.array(golden["spectra"][f"spec_single_{n}_{m}"], np.complex64)
    taps = golden["spectra"][f"taps_{n}_{m}"]
    rng = np.random.default_rng([96, n, ns])
    x = (rng.standard_normal(ns) + 1j * rng.standard_normal(ns)).astype(np.complex64)
    tw, twc = oracle.tables(n, "single")
    l_eff, t0, win_off = oracle.geometry(m, origin, n)
    n_seg = -(-ns // l_eff)
    h0 = taps[:, 0].astype(np.complex64)
    # scale 0.3: float64 product rounded once, like the reference's _store
    out = np.full((3, ns), np.nan, np.complex64)
    for lo, hi in _splits(n_seg):
        K.fused_c2c(x, spectra, tw, twc, m, origin, l_eff, t0, win_off, lo, hi,
                    1, 0.3, h0, out, None, None)
    assert np.array_equal(out, oracle.fused_convolve(
        x, taps, n, origin, "single", pp_kind=1, pp_c=0.3))
    # |y|^2 (fused_c2c_abs2): the reference's float32 re*re + im*im
    y = oracle.fused_convolve(x, taps, n, origin, "single")
    a2 = np.full((3, ns), np.nan, np.float32)
    for lo, hi in _splits(n_seg):
        K.fused_c2c_abs2(x, spectra, tw, twc, m, origin, l_eff, t0, win_off,
                         lo, hi, h0, a2, None, None)
    assert np.array_equal(a2, (y.real * y.real + y.imag * y.imag).astype(np.float32))
    # transforms in place: the exact forward is the reference's dif_fwd
    g = golden["fft"]
    for nn in (8, 256, 2048):
        mat = np.array(g[f"x_{nn}"], dtype=np.complex64, ndmin=2)
        K.dif_fwd_batch(mat, oracle.tables(nn, "single")[0])
        assert np.array_equal(mat[0], g[f"fwd_single_{nn}"])
        inv = np.array(g[f"fwd_single_{nn}"], dtype=np.complex64, ndmin=2)
        K.dit_inv_batch(inv, oracle.tables(nn, "single")[1])
        assert rel_l2_per_filter(inv, g[f"x_{nn}"]) <= 1e-5


@pytest.mark.gpu
def test_fused_r2r_reference_contract():
    """K.fused_r2r with the real taps' rfft bins (natural order, n/2 + 1 --
    transform_filters r2r, ols.py:183-193) over uneven worker ranges."""
    assert has_gpu()
    from paper_1910_01972_b200 import kernels_b200 as K
    n, m, ns, origin = 1024, 257, 20001, 100
    rng = np.random.default_rng([97, n, ns])
    x = rng.standard_normal(ns).astype(np.float32)
    taps = rng.standard_normal((3, m))
    padded = np.zeros((3, n))
    padded[:, :m] = taps
    bins = np.fft.rfft(padded, axis=1).astype(np.complex64)
    l_eff, t0, win_off = oracle.geometry(m, origin, n)
    n_seg = -(-ns // l_eff)
    out = np.full((3, ns), np.nan, np.float32)
    for lo, hi in _splits(n_seg):
        K.fused_r2r(x, bins, None, None, None, None, m, origin, l_eff, t0,
                    win_off, lo, hi, 0, 1.0, taps[:, 0], out, None, None,
                    None, None)
        g_hi = min(hi * l_eff, ns)
        assert np.all(np.isfinite(out[:, :g_hi]))
        assert np.all(np.isnan(out[:, g_hi:]))
    ref = oracle.direct_convolve(x, taps, origin).real
    assert rel_l2_per_filter(out, ref) <= 1e-5


def _global_derivative(y):
    """_store kind 3's global rule: central difference, one-sided at the
    signal ends (_kernels_nb.py:224-262)"""
    d = np.empty_like(y)
    d[:, 1:-1] = 0.5 * (y[:, 2:] - y[:, :-2])
    d[:, 0] = y[:, 1] - y[:, 0]
    d[:, -1] = y[:, -1] - y[:, -2]
    return d


@pytest.mark.gpu
@pytest.mark.parametrize("m", [1, 129])
def test_fused_derivative_reference_contract(m):
    """K.fused_c2c / K.fused_r2r with pp_kind 3 (derivative) over uneven
    worker ranges, called with the reference's own derivative geometry
    (output_windows with halo 1: l_eff = N - M - 1 for M > 1, N - M + 1 with
    t0 = M - 1 for M = 1, ols.py:137-146): only the range's windows are
    written, and the result matches the float64 global derivative."""
    assert has_gpu()
    from paper_1910_01972_b200 import kernels_b200 as K
    n, ns, origin = 512, 9001, m // 2
    rng = np.random.default_rng([98, m])
    halo = 1 if m > 1 else 0
    l_eff = n - m + 1 - 2 * halo
    t0 = m - 1 + halo
    win_off = origin - (m - 1) - halo
    n_seg = -(-ns // l_eff)
    for real in (False, True):
        if real:
            x = rng.standard_normal(ns).astype(np.float32)
            taps = rng.standard_normal((3, m))
            padded = np.zeros((3, n))
            padded[:, :m] = taps
            spec = np.fft.rfft(padded, axis=1).astype(np.complex64)
            out = np.full((3, ns), np.nan, np.float32)
        else:
            x = (rng.standard_normal(ns) + 1j * rng.standard_normal(ns)).astype(np.complex64)
            taps = rng.standard_normal((3, m)) + 1j * rng.standard_normal((3, m))
            spec = np.asarray(oracle.transform_filters(taps, n, "single"),
                              dtype=np.complex64)
            out = np.full((3, ns), np.nan, np.complex64)
        h0 = taps[:, 0]
        for lo, hi in _splits(n_seg):
            if real:
                K.fused_r2r(x, spec, None, None, None, None, m, origin, l_eff,
                            t0, win_off, lo, hi, 3, 1.0, h0, out, None, None,
                            None, None)
            else:
                K.fused_c2c(x, spec, None, None, m, origin, l_eff, t0, win_off,
                            lo, hi, 3, 1.0, h0, out, None, None)
            g_hi = min(hi * l_eff, ns)
            assert np.all(np.isfinite(out[:, :g_hi]))
            assert np.all(np.isnan(out[:, g_hi:]))
        y = oracle.direct_convolve(x, taps, origin)
        ref = _global_derivative(y.real if real else y)
        assert rel_l2_per_filter(out, ref) <= 2e-5, (m, real)
