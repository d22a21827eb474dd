"""GPU parity: the CUDA engine against the reference's own outputs and the
oracle.

Bar (BASELINE.json north_star): per-filter relative L2 <= 1e-5 against the
reference's float64 result for fp32; the reference's own acceptance metric
(relative L-inf, CONV_TOL 1e-4 / 1e-10) is checked alongside.  Fixtures:
tests/golden (produced by the reference itself), plus the C oracle
(oracle/, pinned bit-exact to the reference) for full-size and windowed
checks of configs the fixtures cannot hold.
"""

import numpy as np
import pytest
import torch

import oracle
from cases import CFGS, CONV_GRID, WIN, conv_case_inputs, gen_inputs
from conftest import rel_err, rel_l2_per_filter

pytestmark = pytest.mark.gpu

L2_TOL = 1e-5      # north_star: fp32 per-filter relative L2 vs fp64
LINF_TOL = 1e-4    # reference CONV_TOL single (core.py:32)


@pytest.fixture(scope="module")
def oc():
    import paper_1910_01972_b200 as m
    assert torch.cuda.is_available()
    return m


def _bitrev(n):
    bits = n.bit_length() - 1
    return np.array([int(format(k, f"0{bits}b")[::-1], 2) if bits else 0
                     for k in range(n)])


# ---------------------------------------------------------------------------
# transforms
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("prec", ["single", "double"])
def test_fft_permuted_vs_reference(oc, golden, prec):
    g = golden["fft"]
    P = oc.Precision(prec)
    tol = 2e-6 if prec == "single" else 1e-13
    n = 4
    while n <= 4096:
        p = oc.make_plan(n, "ct_dif_permuted", P)
        x = g[f"x_{n}"].astype(P.complex_dtype)
        fwd = oc.fft_forward_permuted(x, p).cpu().numpy()
        assert rel_err(fwd, g[f"fwd_{prec}_{n}"]) < tol, n
        inv = oc.fft_inverse_permuted(x, p).cpu().numpy()
        assert rel_err(inv, g[f"inv_{prec}_{n}"]) < tol, n
        back = oc.fft_inverse_permuted(oc.fft_forward_permuted(x, p), p)
        assert rel_err(back.cpu().numpy(), x) < tol, n
        n *= 2


def test_fft_known_answers(oc):
    # reference tests/test_fft.py:103-122
    P = oc.Precision.double
    p = oc.make_plan(4, "ct_dif_permuted", P)
    f = lambda v: oc.fft_forward_permuted(v, p).cpu().numpy()  # noqa: E731
    i = lambda v: oc.fft_inverse_permuted(v, p).cpu().numpy()  # noqa: E731
    assert np.allclose(f([1, 0, 0, 0]), np.ones(4))
    assert np.allclose(f([1, 1, 1, 1]), [4, 0, 0, 0])
    assert np.allclose(f([0, 1, 2, 3]), [6, -2, -2 + 2j, -2 - 2j])
    assert np.allclose(i([4, 0, 0, 0]), np.ones(4))
    assert np.allclose(i([6, -2, -2 + 2j, -2 - 2j]), [0, 1, 2, 3])
    with pytest.raises(oc.BadLength):
        oc.fft_forward_permuted(np.zeros(8, complex), p)


def test_fft_vs_naive_dft_all_sizes(oc):
    # acceptance c02: every size against the literal DFT, single <= 1e-5
    for n in [4 << k for k in range(11)]:
        rng = np.random.default_rng([40, n])
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        ref = np.fft.fft(x)
        for prec, tol in (("single", 1e-5), ("double", 1e-12)):
            P = oc.Precision(prec)
            got = oc.fft_forward_permuted(x.astype(P.complex_dtype),
                                          oc.make_plan(n, "ct_dif_permuted", P))
            assert rel_err(got.cpu().numpy()[_bitrev(n)], ref) < tol, (n, prec)


@pytest.mark.parametrize("prec", ["single", "double"])
def test_filter_spectra_vs_reference(oc, golden, prec):
    g = golden["spectra"]
    P = oc.Precision(prec)
    tol = 2e-6 if prec == "single" else 1e-13
    for key in g.files:
        if not key.startswith("taps_"):
            continue
        _, n, m = key.split("_")
        fs = oc.make_filterset(g[key], 0, P)
        p = oc.plan(1000, int(m), "c2c", 0, int(n))
        cached = oc.transform_filters(fs, p, "permuted")
        assert cached.spectra_layout == "permuted" and cached.spectra_n == int(n)
        assert rel_err(cached.spectra.cpu().numpy(),
                       g[f"spec_{prec}_{n}_{m}"]) < tol, key


def test_transform_filters_known_answers(oc):
    # reference tests/test_ols.py:82-98
    P = oc.Precision.double
    fs = oc.make_filterset([[1.0 + 0j, 1.0 + 0j]], 0, P)
    p = oc.plan(100, 2, "c2c", 0, 4)
    assert np.allclose(oc.transform_filters(fs, p, "permuted").spectra[0].cpu(),
                       [2, 0, 1 - 1j, 1 + 1j])
    assert np.allclose(oc.transform_filters(fs, p, "natural").spectra[0].cpu(),
                       [2, 1 - 1j, 0, 1 + 1j])
    delta = oc.make_filterset([[1.0 + 0j]], 0, P)
    for layout in ("natural", "permuted"):
        c = oc.transform_filters(delta, oc.plan(100, 1, "c2c", 0, 8), layout)
        assert np.allclose(c.spectra[0].cpu(), np.ones(8))


def test_natural_spectra_from_engine_fft(oc):
    # "natural" c2c spectra (the comparison variants' layout) come from the
    # engine's in-register FFT read out in natural order: numpy's fft of the
    # zero-padded taps within the fp32 / fp64 transform error
    rng = np.random.default_rng(31)
    for prec, tol in (("single", 2e-6), ("double", 1e-13)):
        P = oc.Precision(prec)
        for n, m in ((4, 3), (64, 17), (1024, 257), (4096, 1000)):
            taps = rng.standard_normal((3, m)) + 1j * rng.standard_normal((3, m))
            fs = oc.transform_filters(oc.make_filterset(taps, 0, P),
                                      oc.plan(5 * n, m, "c2c", 0, n), "natural")
            padded = np.zeros((3, n), np.complex128)
            padded[:, :m] = taps
            want = np.fft.fft(padded, axis=1)
            got = fs.spectra.cpu().numpy()
            assert np.linalg.norm(got - want) / np.linalg.norm(want) <= tol, (prec, n)


# ---------------------------------------------------------------------------
# fused engine vs the reference (golden grid incl. edge cases)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("case", range(len(CONV_GRID)))
def test_fused_vs_reference_grid(oc, golden, case):
    ns, m, nfil, n, origin, _ = CONV_GRID[case]
    x, taps = conv_case_inputs(case)
    g = golden["conv"]
    ref64 = g[f"y_double_{case}"]
    p = oc.plan(ns, m, "c2c", origin, n)
    for prec in ("single", "double"):
        P = oc.Precision(prec)
        sig = oc.make_signal(x, "complex", P)
        fs = oc.make_filterset(taps, origin, P)
        # NaN sentinel: every output index must be written (ols.py:308)
        out = torch.full((nfil, ns), float("nan"), dtype=P.torch_complex,
                         device="cuda")
        y = oc.convolve(sig, fs, p, out=out).cpu().numpy()
        assert np.all(np.isfinite(y)), prec
        if prec == "single":
            assert rel_l2_per_filter(y, ref64) <= L2_TOL
            assert rel_err(y, ref64) <= LINF_TOL
        else:
            assert rel_l2_per_filter(y, ref64) <= 1e-12
            assert rel_err(y, ref64) <= 1e-10
    if f"direct_{case}" in g.files:
        assert rel_err(ref64, g[f"direct_{case}"]) < 1e-10


def test_identity_and_scale_filters(oc):
    # reference test_ols.py:127-135, 179-186
    rng = np.random.default_rng(30)
    x = rng.standard_normal(3000) + 1j * rng.standard_normal(3000)
    P = oc.Precision.double
    sig = oc.make_signal(x, "complex", P)
    out = oc.convolve(sig, oc.make_filterset([[1.0 + 0j]], 0, P),
                      oc.plan(3000, 1, "c2c", 0, 256))
    assert rel_err(out[0].cpu().numpy(), x) < 1e-12
    out = oc.convolve(sig, oc.make_filterset([[2.5 + 0j]], 0, P),
                      oc.plan(3000, 1, "c2c", 0, 64))
    assert rel_err(out[0].cpu().numpy(), 2.5 * x) < 1e-12


def test_scale_postproc_fused(oc):
    x, taps = conv_case_inputs(9)
    ns, m, nfil, n, origin, _ = CONV_GRID[9]
    P = oc.Precision.single
    sig = oc.make_signal(x, "complex", P)
    fs = oc.make_filterset(taps, origin, P)
    p = oc.plan(ns, m, "c2c", origin, n)
    base = oc.convolve(sig, fs, p).cpu().numpy()
    scaled = oc.convolve(sig, fs, p, postproc=oc.PostProcSpec("scale", -1.5))
    assert rel_err(scaled.cpu().numpy(), -1.5 * base) < 1e-6


def test_segment_size_invariance(oc):
    # reference test_ols.py:153-163 / acceptance c04
    rng = np.random.default_rng(32)
    x = rng.standard_normal(4096) + 1j * rng.standard_normal(4096)
    taps = rng.standard_normal((2, 57)) + 1j * rng.standard_normal((2, 57))
    P = oc.Precision.single
    sig = oc.make_signal(x, "complex", P)
    fs = oc.make_filterset(taps, 0, P)
    outs = [oc.convolve(sig, fs, oc.plan(4096, 57, "c2c", 0, n)).cpu().numpy()
            for n in (64, 256, 1024, 4096)]
    for o in outs[1:]:
        assert rel_err(o, outs[0]) < 2e-4


def test_workers_and_ranges_bit_identical(oc):
    # any split of the segment / output range gives identical bits
    # (reference test_ols.py:242-251)
    for case in (12, 18, 19):
        ns, m, nfil, n, origin, _ = CONV_GRID[case]
        x, taps = conv_case_inputs(case)
        P = oc.Precision.single
        sig = oc.make_signal(x, "complex", P)
        fs = oc.transform_filters(oc.make_filterset(taps, origin, P),
                                  oc.plan(ns, m, "c2c", origin, n), "permuted")
        p = oc.plan(ns, m, "c2c", origin, n)
        a = oc.convolve(sig, fs, p, workers=1)
        b = oc.convolve(sig, fs, p, workers=7)
        assert torch.equal(a, b)
        # output-range API over an uneven partition
        from paper_1910_01972_b200.ols import fused_range_launch
        c = torch.full_like(a, float("nan"))
        cuts = [0, 1, ns // 3, ns // 3 + 17, ns - 5, ns]
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            fused_range_launch(sig.samples, 0, ns, fs.spectra_dev, nfil, p, lo,
                               hi, oc.NONE, c, ns, 0, P)
        assert torch.equal(a, c)


def test_host_streaming_path_bit_identical(oc):
    ns, m, nfil, n, origin, _ = CONV_GRID[18]
    x, taps = conv_case_inputs(18)
    P = oc.Precision.single
    p = oc.plan(ns, m, "c2c", origin, n)
    fs = oc.transform_filters(oc.make_filterset(taps, origin, P), p, "permuted")
    dev = oc.convolve(oc.make_signal(x, "complex", P), fs, p)
    hsig = oc.make_signal(torch.from_numpy(x.astype(np.complex64)).pin_memory(),
                          "complex", P, device="cpu")
    host_out = torch.empty((nfil, ns), dtype=torch.complex64).pin_memory()
    got = oc.convolve(hsig, fs, p, out=host_out, chunk_segments=2)
    assert got.data_ptr() == host_out.data_ptr()
    assert torch.equal(host_out, dev.cpu())


@pytest.mark.parametrize("mode,nfil", [("c2c", 3), ("c2c", 7), ("c2c", 16),
                                       ("r2r", 7)])
def test_host_streaming_filter_chunks_bit_identical(oc, mode, nfil):
    # default host path: chunks of whole output rows (filters), one
    # contiguous D2H each; ragged last chunk for nfil = 7 / 16
    from paper_1910_01972_b200 import ols as ols_mod
    ns, m, n, origin = 50000, 77, 512, 3
    rng = np.random.default_rng([71, nfil])
    real = mode == "r2r"
    x = rng.standard_normal(ns) + (0 if real else 1j * rng.standard_normal(ns))
    taps = rng.standard_normal((nfil, m)) + (
        0 if real else 1j * rng.standard_normal((nfil, m)))
    P = oc.Precision.single
    kind = "real" if real else "complex"
    hdt = np.float32 if real else np.complex64
    tdt = torch.float32 if real else torch.complex64
    p = oc.plan(ns, m, mode, origin, n)
    fs = oc.transform_filters(oc.make_filterset(taps, origin, P), p,
                              "natural" if real else "permuted")
    dev = oc.convolve(oc.make_signal(x, kind, P), fs, p)
    hsig = oc.make_signal(torch.from_numpy(x.astype(hdt)).pin_memory(),
                          kind, P, device="cpu")
    host_out = torch.full((nfil, ns), float("nan"), dtype=tdt).pin_memory()
    tile = ols_mod._STREAM_TILE
    try:
        # a small tile forces several row chunks (2 rows per chunk)
        ols_mod._STREAM_TILE = 2 * ns * host_out.element_size()
        oc.convolve(hsig, fs, p, out=host_out)
    finally:
        ols_mod._STREAM_TILE = tile
    assert torch.equal(host_out, dev.cpu())


def test_spectra_handed_over_in_reference_layout(oc, golden):
    # a FilterSet whose permuted cache was filled elsewhere (e.g. by the
    # reference) is converted to the engine layout once
    g = golden["spectra"]
    taps = g["taps_2048_400"]
    P = oc.Precision.single
    fs = oc.make_filterset(taps, 0, P)
    p = oc.plan(9000, 400, "c2c", 0, 2048)
    spec = torch.from_numpy(g["spec_single_2048_400"]).cuda()
    handed = fs.with_spectra(spec, "permuted", 2048)
    rng = np.random.default_rng(5)
    x = rng.standard_normal(9000) + 1j * rng.standard_normal(9000)
    sig = oc.make_signal(x, "complex", P)
    a = oc.convolve(sig, handed, p).cpu().numpy()
    b = oc.convolve(sig, fs, p).cpu().numpy()
    assert rel_l2_per_filter(a, b) < 1e-6


def test_variants_agree(oc):
    # reference test_ols.py:166-176 (pipelined = the cuFFT-OLS comparison
    # point, full_fft_baseline, direct_oracle)
    rng = np.random.default_rng(33)
    x = rng.standard_normal(6000) + 1j * rng.standard_normal(6000)
    taps = rng.standard_normal((3, 65)) + 1j * rng.standard_normal((3, 65))
    P = oc.Precision.double
    sig = oc.make_signal(x, "complex", P)
    fs = oc.make_filterset(taps, 32, P)
    p = oc.plan(6000, 65, "c2c", 32, 512)
    fused = oc.convolve(sig, fs, p).cpu().numpy()
    for v in ("pipelined", "full_fft_baseline", "direct_oracle"):
        assert rel_err(oc.convolve(sig, fs, p, variant=v).cpu().numpy(),
                       fused) < 1e-10, v


def test_cufft_callback_ols_vs_reference(oc, golden):
    """variant="cufft_ols" (the paper's cuFFT-based OLS comparison point:
    batched C2C over overlapping windows, multiply kernel, batched inverse,
    discard kernel, on L2-sized chunks) on every c2c golden cell: within the
    fp32 bar of the reference's float64 result; also the cfg3 shape at a
    larger size (several segment chunks), and scale."""
    g = golden["conv"]
    P = oc.Precision.single
    for i, (ns, m, nfil, n, origin, real_taps) in enumerate(CONV_GRID):
        x, taps = conv_case_inputs(i)
        p = oc.plan(ns, m, "c2c", origin, n)
        out = torch.full((nfil, ns), float("nan"), dtype=torch.complex64,
                         device="cuda")
        y = oc.convolve(oc.make_signal(x, "complex", P),
                        oc.make_filterset(taps, origin, P), p,
                        variant="cufft_ols", out=out).cpu().numpy()
        assert np.all(np.isfinite(y)), i        # every output written once
        assert rel_l2_per_filter(y, g[f"y_double_{i}"]) <= L2_TOL, i
    ns, m, nfil, n = 300_000, 400, 4, 2048
    rng = np.random.default_rng([98, ns])
    x = rng.standard_normal(ns) + 1j * rng.standard_normal(ns)
    taps = rng.standard_normal((nfil, m)) + 1j * rng.standard_normal((nfil, m))
    p = oc.plan(ns, m, "c2c", 0, n)
    y = oc.convolve(oc.make_signal(x, "complex", P),
                    oc.make_filterset(taps, 0, P), p,
                    variant="cufft_ols",
                    postproc=oc.PostProcSpec("scale", 0.5)).cpu().numpy()
    ref = 0.5 * oracle.direct_convolve(x, taps, 0)
    assert rel_l2_per_filter(y, ref) <= L2_TOL


def test_error_detection(oc):
    # reference test_ols.py:189-221
    rng = np.random.default_rng(36)
    P = oc.Precision.single
    sig = oc.make_signal(rng.standard_normal(500) + 0j, "complex", P)
    fs = oc.make_filterset(rng.standard_normal((1, 9)) + 1j, 0, P)
    p = oc.plan(500, 9, "c2c", 0, 64)
    natural = oc.transform_filters(fs, p, "natural")
    with pytest.raises(oc.LayoutMismatch):
        oc.convolve(sig, natural, p, variant="fused")
    permuted = oc.transform_filters(fs, p, "permuted")
    with pytest.raises(oc.LayoutMismatch):
        oc.convolve(sig, permuted, p, variant="pipelined")
    with pytest.raises(oc.PlanMismatch):
        oc.convolve(sig, permuted, oc.plan(500, 9, "c2c", 0, 128))
    with pytest.raises(oc.PlanMismatch):
        oc.convolve(oc.make_signal(np.ones(400) + 0j, "complex", P), fs, p)
    with pytest.raises(oc.PlanMismatch):
        oc.convolve(oc.make_signal(np.ones(500) + 0j, "complex",
                                   oc.Precision.double), fs, p)
    with pytest.raises(oc.PlanMismatch):
        oc.convolve(sig, oc.make_filterset(np.ones((1, 9)) + 0j, 3, P), p)
    with pytest.raises(oc.EmptyInput):
        oc.make_signal([], "complex")
    with pytest.raises(oc.RaggedFilters):
        oc.make_filterset([[1, 2], [1]])
    with pytest.raises(oc.BadOrigin):
        oc.make_filterset([[1, 2]], 2)


# ---------------------------------------------------------------------------
# BASELINE.json configs at full size
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("cfg", [c[0] for c in CFGS])
def test_baseline_configs_full_size_windows(oc, golden, cfg):
    """cfg1-cfg4 at their full sizes: fixed windows (both signal ends, segment
    seams, interior) against the reference's float64 output, plus per-filter
    checksums of the whole output (sum |y|^2, sum y)."""
    g = golden["cfg"]
    ns, m, nfil, n = (int(v) for v in g[f"{cfg}_params"])
    x, taps = gen_inputs(ns, m, nfil)
    P = oc.Precision.single
    p = oc.plan(ns, m, "c2c", 0, n)
    sig = oc.make_signal(x, "complex", P)
    fs = oc.transform_filters(oc.make_filterset(taps, 0, P), p, "permuted")
    y = oc.convolve(sig, fs, p)
    starts = g[f"{cfg}_starts"]
    win = torch.stack([y[:, s:s + WIN] for s in starts], dim=1).cpu().numpy()
    ref = g[f"{cfg}_win"].astype(np.complex128)
    assert rel_l2_per_filter(win.reshape(nfil, -1), ref.reshape(nfil, -1)) <= L2_TOL
    sumsq = (y.abs().double() ** 2).sum(dim=1).cpu().numpy()
    assert np.max(np.abs(sumsq / g[f"{cfg}_sumsq"] - 1)) < 2e-6
    ssum = y.to(torch.complex128).sum(dim=1).cpu().numpy()
    assert np.max(np.abs(ssum - g[f"{cfg}_sum"]) /
                  np.sqrt(g[f"{cfg}_sumsq"])) < 1e-5


def test_fdas_full_output_vs_oracle(oc):
    """cfg3 (FDAS: 2^23 x 96 filters, M=400, N=2048), every output sample:
    per-filter relative L2 against the oracle's float64 fused result."""
    ns, m, nfil, n = 1 << 23, 400, 96, 2048
    x, taps = gen_inputs(ns, m, nfil)
    P = oc.Precision.single
    p = oc.plan(ns, m, "c2c", 0, n)
    y = oc.convolve(oc.make_signal(x, "complex", P),
                    oc.transform_filters(oc.make_filterset(taps, 0, P), p,
                                         "permuted"), p).cpu().numpy()
    ref = oracle.fused_convolve(x, taps, n, 0, "double")
    err = rel_l2_per_filter(y, ref)
    assert err <= L2_TOL, err
    assert rel_err(y, ref) <= LINF_TOL


def test_cfg5_geometry_windows_vs_oracle(oc):
    """cfg5 (2^30 samples, 64 filters, M=512, N=4096): the full output is
    512 GiB, so outputs are produced for windows (signal start, a shard seam,
    interior, signal end) through the range API and compared with the
    oracle's direct float64 convolution of the same windows."""
    ns, m, nfil, n = 1 << 30, 512, 64, 4096
    gen = torch.Generator(device="cuda").manual_seed(0)
    xs = torch.randn(ns, dtype=torch.complex64, device="cuda", generator=gen)
    rng = np.random.default_rng([0, ns, m, nfil, 0, 0])
    taps = rng.standard_normal((nfil, m)) + 1j * rng.standard_normal((nfil, m))
    P = oc.Precision.single
    p = oc.plan(ns, m, "c2c", 0, n)
    fs = oc.transform_filters(oc.make_filterset(taps, 0, P), p, "permuted")
    sig = oc.Signal(samples=xs, length=ns, domain="time", value_kind="complex")
    from paper_1910_01972_b200.ols import fused_range_launch
    for a in (0, ns // 2 - 100, 3 * (ns // 8) + 12345, ns - 300):
        b = a + 300
        out = torch.empty((nfil, b - a), dtype=torch.complex64, device="cuda")
        fused_range_launch(sig.samples, 0, ns, fs.spectra_dev, nfil, p, a, b,
                           oc.NONE, out, b - a, a, P)
        lo, hi = max(0, a - (m - 1)), b
        xw = xs[lo:hi].cpu().numpy().astype(np.complex128)
        full = np.zeros(hi - (a - (m - 1)), np.complex128)
        full[lo - (a - (m - 1)):] = xw
        ref = oracle.direct_window(full, taps, 0, m - 1, m - 1 + (b - a))
        assert rel_l2_per_filter(out.cpu().numpy(), ref) <= L2_TOL, a


def test_cfg5_shard_seams_from_halo_buffers(oc):
    """cfg5 sharded over G = 2, 4, 8 ranks: every rank's persistent halo'd
    buffer (sharding.HaloBuffer, halos filled as the transport would) alone
    produces the outputs at both ends of its shard -- through the chunked
    shard engine (convolve_shard_chunked) -- bit-identical to the unsharded
    launch over the global signal and within the fp32 bar of the oracle."""
    from paper_1910_01972_b200.ols import fused_range_launch
    from paper_1910_01972_b200.sharding import (HaloBuffer,
                                                convolve_shard_chunked,
                                                make_shards)
    ns, m, nfil, n = 1 << 30, 512, 64, 4096
    gen = torch.Generator(device="cuda").manual_seed(1)
    xs = torch.randn(ns, dtype=torch.complex64, device="cuda", generator=gen)
    rng = np.random.default_rng([0, ns, m, nfil, 0, 0])
    taps = rng.standard_normal((4, m)) + 1j * rng.standard_normal((4, m))
    P = oc.Precision.single
    p = oc.plan(ns, m, "c2c", 0, n)
    fs = oc.transform_filters(oc.make_filterset(taps, 0, P), p, "permuted")
    w = 300
    tile = torch.empty((4, w), dtype=torch.complex64, device="cuda")
    for world in (2, 4, 8):
        shards = make_shards(p, world)
        for r, sh in enumerate(shards):
            hb = HaloBuffer(shards, r, torch.complex64, "cuda")
            hb.own.copy_(xs[sh.g_lo:sh.g_hi])
            hb.fill_from(xs)
            for a in (sh.g_lo, sh.g_hi - w):
                seg = type(sh)(sh.rank, sh.world, a, a + w, sh.x_lo, sh.x_hi)
                got = {}
                convolve_shard_chunked(
                    hb.buffer, seg, p, fs.spectra_dev, 4, P, tile,
                    sink=lambda ga, gb, t: got.setdefault(ga, t.clone()))
                want = torch.empty((4, w), dtype=torch.complex64, device="cuda")
                fused_range_launch(xs, 0, ns, fs.spectra_dev, 4, p, a, a + w,
                                   oc.NONE, want, w, a, P)
                assert torch.equal(got[a], want), (world, r, a)
                lo = max(0, a - (m - 1))
                xw = xs[lo:a + w].cpu().numpy().astype(np.complex128)
                full = np.zeros(a + w - (a - (m - 1)), np.complex128)
                full[lo - (a - (m - 1)):] = xw
                ref = oracle.direct_window(full, taps, 0, m - 1, m - 1 + w)
                assert rel_l2_per_filter(got[a].cpu().numpy(), ref) <= L2_TOL
            del hb


@pytest.mark.parametrize("mode", ["c2c", "r2r"])
def test_beyond_int32_sample_indices_vs_oracle(oc, mode):
    """N_s = 2^31 + 12345 samples (c2c: 17 GB in, 17 GB out): every sample
    and output index crosses the int32 range.  Windows around 2^31, at the
    end and at the start are compared with the oracle's direct float64
    convolution; the full output is checked for coverage (no NaN left)."""
    ns, m, nfil, n, origin = (1 << 31) + 12345, 64, 1, 1024, 5
    real = mode == "r2r"
    gen = torch.Generator(device="cuda").manual_seed(3)
    xs = torch.randn(ns, dtype=torch.float32 if real else torch.complex64,
                     device="cuda", generator=gen)
    rng = np.random.default_rng([3, m, nfil])
    taps = rng.standard_normal((nfil, m)) + (
        0 if real else 1j * rng.standard_normal((nfil, m)))
    P = oc.Precision.single
    p = oc.plan(ns, m, mode, origin, n)
    fs = oc.transform_filters(oc.make_filterset(taps, origin, P), p,
                              "natural" if real else "permuted")
    sig = oc.Signal(samples=xs, length=ns, domain="time",
                    value_kind="real" if real else "complex")
    out = torch.full((nfil, ns), float("nan"), dtype=xs.dtype, device="cuda")
    oc.convolve(sig, fs, p, out=out)
    assert not torch.isnan(out).any()
    for a in (0, (1 << 31) - 150, (1 << 31) + 7, ns - 300):
        b = min(a + 300, ns)
        # y[g] = sum_k h[k] x[g - k + origin]
        lo, hi = a - (m - 1) + origin, b + origin
        full = np.zeros(hi - lo, np.complex128)
        clo, chi = max(lo, 0), min(hi, ns)
        full[clo - lo:chi - lo] = xs[clo:chi].cpu().numpy()
        ref = oracle.direct_window(full, taps, 0, m - 1, m - 1 + (b - a))
        got = out[:, a:b].cpu().numpy()
        assert rel_l2_per_filter(got, ref) <= L2_TOL, a
    del out, xs
    torch.cuda.empty_cache()


# ---- exact mode: the reference's arithmetic, bit for bit -------------------

@pytest.mark.parametrize("prec", ["single", "double"])
def test_fused_exact_bit_identical_to_reference(oc, golden, prec):
    """variant="fused_exact" reproduces the reference's own fp32 / fp64
    convolve(variant="fused") outputs bit for bit on every cell of the
    golden grid (first/last segment, M = 1, M = N, N_s < L, origin > 0,
    real taps on a complex signal, N = 4 .. 4096)."""
    g = golden["conv"]
    P = oc.Precision.single if prec == "single" else oc.Precision.double
    for i, (ns, m, nfil, n, origin, _) in enumerate(CONV_GRID):
        x, taps = conv_case_inputs(i)
        p = oc.plan(ns, m, "c2c", origin, n)
        y = oc.convolve(oc.make_signal(x, "complex", P),
                        oc.make_filterset(taps, origin, P), p,
                        variant="fused_exact")
        ref = torch.from_numpy(g[f"y_{prec}_{i}"])
        assert torch.equal(y.cpu(), ref), (prec, i)


def test_fused_exact_scale_abs2_and_workers(oc):
    """Exact mode with postproc scale (the reference oracle, itself pinned
    bit-exact to the reference) and magnitude_squared, split over workers."""
    ns, m, nfil, n, origin = 20000, 129, 3, 512, 7
    rng = np.random.default_rng([72, ns])
    x = rng.standard_normal(ns) + 1j * rng.standard_normal(ns)
    taps = rng.standard_normal((nfil, m)) + 1j * rng.standard_normal((nfil, m))
    P = oc.Precision.single
    p = oc.plan(ns, m, "c2c", origin, n)
    sig = oc.make_signal(x, "complex", P)
    fs = oc.make_filterset(taps, origin, P)
    ys = oc.convolve(sig, fs, p, variant="fused_exact",
                     postproc=oc.PostProcSpec("scale", 0.3), workers=3)
    ref = oracle.fused_convolve(x, taps, n, origin, "single", pp_kind=1,
                                pp_c=0.3)
    assert torch.equal(ys.cpu(), torch.from_numpy(ref))
    y = oc.convolve(sig, fs, p, variant="fused_exact")
    a2 = oc.convolve(sig, fs, p, variant="fused_exact",
                     postproc=oc.PostProcSpec("magnitude_squared"))
    yc = y.cpu().numpy()
    want = yc.real * yc.real + yc.imag * yc.imag   # float32, no FMA
    assert np.array_equal(a2.cpu().numpy(), want.astype(np.float32))


def test_fused_exact_scale_bit_identical_to_reference(oc, golden):
    """Exact mode with postproc scale 0.3 equals the reference's own fp32 and
    fp64 outputs (pp_cases.npz, made by the reference) bit for bit: pp_c is
    applied in float64 and rounded once, as the reference's _store does."""
    from cases import PP_GRID, pp_case_inputs, pp_scale
    cells = [i for i, c in enumerate(PP_GRID) if c[5] == "c2c" and c[6] == "scale"]
    assert cells
    for i in cells:
        ns, m, nfil, n, origin, _, _ = PP_GRID[i]
        x, taps = pp_case_inputs(i)
        p = oc.plan(ns, m, "c2c", origin, n)
        for prec in ("single", "double"):
            P = oc.Precision(prec)
            y = oc.convolve(oc.make_signal(x, "complex", P),
                            oc.make_filterset(taps, origin, P), p,
                            variant="fused_exact",
                            postproc=oc.PostProcSpec("scale", pp_scale(i)),
                            workers=2)
            ref = torch.from_numpy(golden["pp"][f"y_{prec}_{i}"])
            assert torch.equal(y.cpu(), ref), (i, prec)


def test_fused_exact_host_streaming(oc, golden):
    """Exact mode from a pinned host signal into a pinned host output (row
    chunks, contiguous D2H) equals the reference's fp32 output bit for bit."""
    g = golden["conv"]
    from paper_1910_01972_b200 import ols as ols_mod
    for i in (10, 17, 18):
        ns, m, nfil, n, origin, _ = CONV_GRID[i]
        x, taps = conv_case_inputs(i)
        P = oc.Precision.single
        p = oc.plan(ns, m, "c2c", origin, n)
        hsig = oc.make_signal(
            torch.from_numpy(x.astype(np.complex64)).pin_memory(), "complex",
            P, device="cpu")
        host = torch.full((nfil, ns), float("nan"),
                          dtype=torch.complex64).pin_memory()
        tile = ols_mod._STREAM_TILE
        try:
            ols_mod._STREAM_TILE = ns * 8      # one row per chunk
            oc.convolve(hsig, oc.make_filterset(taps, origin, P), p,
                        variant="fused_exact", out=host)
        finally:
            ols_mod._STREAM_TILE = tile
        assert torch.equal(host, torch.from_numpy(g[f"y_single_{i}"])), i
