"""GPU parity of the real (r2r) fused path and the magnitude_squared and
derivative epilogues against the reference's own outputs
(tests/golden/pp_cases.npz, made by the reference's fused_r2r /
fused_c2c_abs2 and pinned against the oracle in test_oracle.py).

The engine transforms two real segments as one complex segment (re / im), so
the tests also cover odd segment counts, range splits that start on the
second segment of a pair, and the host streaming path.
"""

import numpy as np
import pytest
import torch

from cases import PP_GRID, pp_case_inputs, pp_scale
from conftest import rel_err, rel_l2_per_filter

pytestmark = pytest.mark.gpu

L2_TOL = 1e-5


@pytest.fixture(scope="module")
def oc():
    import paper_1910_01972_b200 as m
    assert torch.cuda.is_available()
    return m


def _run(oc, case, prec, out=None, workers=1, layout="natural"):
    ns, m, nfil, n, origin, mode, ppk = PP_GRID[case]
    x, taps = pp_case_inputs(case)
    P = oc.Precision(prec)
    vk = "real" if mode == "r2r" else "complex"
    p = oc.plan(ns, m, mode, origin, n)
    pp = oc.PostProcSpec(ppk, pp_scale(case))
    fs = oc.transform_filters(oc.make_filterset(taps, origin, P), p,
                              "natural" if mode == "r2r" else "permuted")
    return oc.convolve(oc.make_signal(x, vk, P), fs, p, postproc=pp, out=out,
                       workers=workers), p, fs


@pytest.mark.parametrize("case", range(len(PP_GRID)))
def test_real_path_and_abs2_vs_reference(oc, golden, case):
    ns, m, nfil, n, origin, mode, ppk = PP_GRID[case]
    ref = golden["pp"][f"y_double_{case}"]
    for prec in ("single", "double"):
        P = oc.Precision(prec)
        real = mode == "r2r" or ppk == "magnitude_squared"
        out = torch.full((nfil, ns), float("nan"),
                         dtype=P.torch_real if real else P.torch_complex,
                         device="cuda")
        y, _, _ = _run(oc, case, prec, out=out)
        y = y.cpu().numpy()
        assert np.isrealobj(y) == real
        assert np.all(np.isfinite(y)), prec   # every output written once
        tol_l2, tol_inf = (L2_TOL, 1e-4) if prec == "single" else (1e-12, 1e-10)
        if ppk in ("magnitude_squared", "derivative"):
            # squares double the relative error; differences of neighbours
            # amplify it by up to ~2 (cancellation)
            tol_l2, tol_inf = 2 * tol_l2, 2 * tol_inf
        assert rel_l2_per_filter(y, ref) <= tol_l2, prec
        assert rel_err(y, ref) <= tol_inf, prec


def test_r2r_splits_bit_identical(oc):
    # workers, output-range cuts at odd segment boundaries (second half of a
    # segment pair) and the host streaming path all give the same bits
    from paper_1910_01972_b200.ols import fused_range_launch
    for case in (7, 8, 10):
        ns, m, nfil, n, origin, mode, ppk = PP_GRID[case]
        a, p, fs = _run(oc, case, "single")
        b, _, _ = _run(oc, case, "single", workers=5)
        assert torch.equal(a, b)
        x, _ = pp_case_inputs(case)
        P = oc.Precision.single
        sig = oc.make_signal(x, "real", P)
        pp = oc.PostProcSpec(ppk, pp_scale(case))
        le = p.valid_len
        c = torch.full_like(a, float("nan"))
        cuts = [0, 1, le + 3, 3 * le, 3 * le + 1, ns // 2, ns - 2, ns]
        cuts = sorted(set(min(max(v, 0), ns) for v in cuts))
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            fused_range_launch(sig.samples, 0, ns, fs.spectra_dev, nfil, p, lo,
                               hi, pp, c, ns, 0, P)
        assert torch.equal(a, c)
        hsig = oc.make_signal(torch.from_numpy(x.astype(np.float32)).pin_memory(),
                              "real", P, device="cpu")
        host = torch.empty((nfil, ns), dtype=torch.float32).pin_memory()
        oc.convolve(hsig, fs, p, postproc=pp, out=host, chunk_segments=3)
        assert torch.equal(host, a.cpu())


def test_r2r_vs_cufft_pipelined_and_direct(oc):
    # the cuFFT comparison point (R2C / C2R) and the direct oracle variant
    case = 7
    a, p, fs = _run(oc, case, "single")
    ns, m, nfil, n, origin, mode, ppk = PP_GRID[case]
    x, taps = pp_case_inputs(case)
    P = oc.Precision.single
    sig = oc.make_signal(x, "real", P)
    b = oc.convolve(sig, fs, p, variant="pipelined")
    d = oc.convolve(sig, oc.make_filterset(taps, origin, P), p,
                    variant="direct_oracle")
    assert b.dtype == torch.float32 and d.dtype == torch.float32
    assert rel_err(a.cpu().numpy(), d.cpu().numpy()) < 1e-5
    assert rel_err(b.cpu().numpy(), d.cpu().numpy()) < 1e-5


def test_fdas_shape_real_full_output_vs_oracle(oc):
    # cfg3 geometry on the real path at 2^20 samples, every output checked
    import oracle
    ns, m, nfil, n = 1 << 20, 400, 8, 2048
    rng = np.random.default_rng([50, ns, m, nfil])
    x = rng.standard_normal(ns)
    taps = rng.standard_normal((nfil, m))
    P = oc.Precision.single
    p = oc.plan(ns, m, "r2r", 0, n)
    fs = oc.transform_filters(oc.make_filterset(taps, 0, P), p, "natural")
    y = oc.convolve(oc.make_signal(x, "real", P), fs, p).cpu().numpy()
    ref = oracle.direct_convolve(x, taps, 0).real
    assert rel_l2_per_filter(y, ref) <= L2_TOL


@pytest.mark.parametrize("mode", ["c2c", "r2r"])
def test_autotune_segment_size(oc, mode):
    # ols.py:471-526: feasible power-of-two candidates >= max(M, floor),
    # fastest wins; infeasible candidates are dropped
    times = oc.measure_segment_times(100, mode, [32, 128, 256, 1024, 3000],
                                     probe_len=1 << 16, n_filters=2)
    assert sorted(times) == [128, 256, 1024]
    assert all(t > 0 for t in times.values())
    best = oc.autotune_segment_size(100, mode, [128, 256, 1024],
                                    probe_len=1 << 16, n_filters=2)
    assert best in (128, 256, 1024)
    with pytest.raises(oc.SegmentTooSmall):
        oc.measure_segment_times(100, mode, [16, 64])


@pytest.mark.parametrize("mode", ["c2c", "r2r"])
def test_sharded_outputs_bit_identical(oc, mode):
    # every rank's launch from its own halo'd input slice (make_shards +
    # convolve_shard, the multi-GPU data path without the transport) equals
    # the single-call result bit for bit; r2r extents are pair-aligned; the
    # derivative's extents (make_shards(postproc=...)) carry its halo
    from paper_1910_01972_b200.sharding import convolve_shard, make_shards
    ns, m, nfil, n, origin = 20000, 400, 3, 2048, 17
    rng = np.random.default_rng([60, ns])
    real = mode == "r2r"
    x = rng.standard_normal(ns) if real else (rng.standard_normal(ns)
                                              + 1j * rng.standard_normal(ns))
    taps = rng.standard_normal((nfil, m)) if real else (
        rng.standard_normal((nfil, m)) + 1j * rng.standard_normal((nfil, m)))
    P = oc.Precision.single
    p = oc.plan(ns, m, mode, origin, n)
    fs = oc.transform_filters(oc.make_filterset(taps, origin, P), p,
                              "natural" if real else "permuted")
    sig = oc.make_signal(x, "real" if real else "complex", P)
    for pp in (None, oc.PostProcSpec("derivative")):
        full = oc.convolve(sig, fs, p, postproc=pp)
        for world in (2, 3, 5):
            got = torch.full_like(full, float("nan"))
            for sh in make_shards(p, world, postproc=pp):
                if sh.g_hi <= sh.g_lo:
                    continue
                xl = sig.samples[sh.x_lo:sh.x_hi].clone()   # this rank's data
                got[:, sh.g_lo:sh.g_hi] = convolve_shard(xl, sh, p, fs,
                                                         postproc=pp)
            assert torch.equal(got, full), (world, pp)


_VARIANT_SCRIPT = r"""
import sys, numpy as np
sys.path[:0] = [{root!r}, {golden!r}]
import paper_1910_01972_b200 as oc
from cases import CONV_GRID, conv_case_inputs
g = np.load({npz!r})
worst = 0.0
for case in (12, 13, 17, 18, 19):
    ns, m, nfil, n, origin, _ = CONV_GRID[case]
    x, taps = conv_case_inputs(case)
    P = oc.Precision.single
    y = oc.convolve(oc.make_signal(x, "complex", P),
                    oc.make_filterset(taps, origin, P),
                    oc.plan(ns, m, "c2c", origin, n)).cpu().numpy()
    ref = g[f"y_double_{{case}}"]
    e = np.max(np.linalg.norm(y - ref, axis=1) / np.linalg.norm(ref, axis=1))
    worst = max(worst, e)
print(worst)
"""


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 8])
def test_tuning_variants_correct(variant):
    # the OLSB_VARIANT kernel policies (tuning sweeps) produce correct results
    # (variants 4-7 are ablations and intentionally wrong)
    import os
    import subprocess
    import sys
    from conftest import GOLDEN, ROOT
    code = _VARIANT_SCRIPT.format(root=ROOT, golden=GOLDEN,
                                  npz=os.path.join(GOLDEN, "conv_cases.npz"))
    env = dict(os.environ, OLSB_VARIANT=str(variant))
    res = subprocess.run([sys.executable, "-c", code], env=env,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    assert float(res.stdout.strip().splitlines()[-1]) <= L2_TOL


@pytest.mark.parametrize("mode,ppk", [("c2c", "none"), ("c2c", "scale"),
                                      ("c2c", "magnitude_squared"),
                                      ("c2c", "derivative"), ("r2r", "none"),
                                      ("r2r", "derivative")])
def test_executor_and_graph_replay_bit_identical(oc, mode, ppk):
    ns, m, nfil, n, origin = 30000, 129, 3, 1024, 5
    rng = np.random.default_rng([70, ns])
    real = mode == "r2r"
    x = rng.standard_normal(ns) if real else (rng.standard_normal(ns)
                                              + 1j * rng.standard_normal(ns))
    taps = rng.standard_normal((nfil, m)) if real else (
        rng.standard_normal((nfil, m)) + 1j * rng.standard_normal((nfil, m)))
    P = oc.Precision.single
    p = oc.plan(ns, m, mode, origin, n)
    pp = oc.PostProcSpec(ppk, 0.5 if ppk == "scale" else 1.0)
    fs = oc.make_filterset(taps, origin, P)
    sig = oc.make_signal(x, "real" if real else "complex", P)
    ref = oc.convolve(sig, fs, p, postproc=pp)
    ex = oc.Executor(fs, p, pp)
    assert torch.equal(ex(sig), ref)
    out = torch.empty_like(ref)
    xs = sig.samples.clone()
    run = ex.graph(xs, out)
    run()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    # new data through the same captured graph
    xs.mul_(2)
    run()
    torch.cuda.synchronize()
    want = oc.convolve(oc.make_signal(xs, "real" if real else "complex", P), fs,
                       p, postproc=pp)
    assert torch.equal(out, want)
    with pytest.raises(ValueError):
        ex(sig.samples[:-1])


def test_streaming_small_n_filter_chunks(oc):
    """Host streaming in row chunks whose spectra start at a filter offset
    that is not texture-aligned (N = 16: 128-byte rows): the engine binds the
    aligned-down base and offsets its fetches.  Bit-identical to the device
    path, for c2c, c2c magnitude_squared and r2r."""
    ns, m, nfil, n = 5000, 9, 7, 16
    rng = np.random.default_rng([91, ns, nfil])
    x = rng.standard_normal(ns) + 1j * rng.standard_normal(ns)
    taps = rng.standard_normal((nfil, m)) + 1j * rng.standard_normal((nfil, m))
    P = oc.Precision.single
    for mode, ppk in (("c2c", "none"), ("c2c", "magnitude_squared"),
                      ("r2r", "none")):
        xs = x if mode == "c2c" else x.real
        ts = taps if mode == "c2c" else taps.real
        vk = "complex" if mode == "c2c" else "real"
        p = oc.plan(ns, m, mode, 0, n)
        fs = oc.transform_filters(oc.make_filterset(ts, 0, P), p,
                                  "permuted" if mode == "c2c" else "natural")
        pp = oc.PostProcSpec(ppk)
        dev = oc.convolve(oc.make_signal(xs, vk, P), fs, p, postproc=pp)
        host = torch.full(tuple(dev.shape), float("nan"),
                          dtype=dev.dtype).pin_memory()
        hsig = oc.make_signal(torch.from_numpy(np.ascontiguousarray(xs).astype(
            np.complex64 if mode == "c2c" else np.float32)).pin_memory(),
            vk, P, device="cpu")
        oc.convolve(hsig, fs, p, postproc=pp, out=host)
        assert torch.equal(host, dev.cpu()), (mode, ppk)


def test_comparison_variants_fill_out(oc):
    """direct_oracle / full_fft_baseline write a caller-provided `out`."""
    ns, m, nfil, n = 3000, 17, 2, 64
    rng = np.random.default_rng([92, ns])
    x = rng.standard_normal(ns) + 1j * rng.standard_normal(ns)
    taps = rng.standard_normal((nfil, m)) + 1j * rng.standard_normal((nfil, m))
    P = oc.Precision.single
    p = oc.plan(ns, m, "c2c", 0, n)
    sig = oc.make_signal(x, "complex", P)
    fs = oc.make_filterset(taps, 0, P)
    for variant in ("direct_oracle", "full_fft_baseline"):
        out = torch.full((nfil, ns), float("nan"), dtype=torch.complex64,
                         device="cuda")
        y = oc.convolve(sig, fs, p, variant=variant, out=out)
        assert y is out and torch.isfinite(torch.view_as_real(out)).all()
        ref = oc.convolve(sig, fs, p, variant=variant)
        assert torch.equal(out, ref)


def test_r2r_spectra_from_engine_fft(oc):
    """transform_filters on the real path: the packed rfft bins (n/2 + 1,
    natural order, the reference's semantics, ols.py:183-193) come out of
    the engine's own FFT (no cuFFT), together with the engine layout."""
    rng = np.random.default_rng([99])
    for n, m in ((8, 3), (1024, 257), (4096, 1025)):
        taps = rng.standard_normal((3, m))
        p = oc.plan(10_000, m, "r2r", 0, n)
        fs = oc.transform_filters(oc.make_filterset(taps, 0, oc.Precision.single),
                                  p, "natural")
        assert fs.spectra.shape == (3, n // 2 + 1) and fs.spectra_dev is not None
        padded = np.zeros((3, n))
        padded[:, :m] = taps
        want = np.fft.rfft(padded, axis=1)
        assert rel_l2_per_filter(fs.spectra.cpu().numpy(), want) <= 1e-6, n


@pytest.mark.parametrize("mode", ["c2c", "r2r"])
@pytest.mark.parametrize("m", [1, 65])
def test_derivative_streaming_and_ranges(oc, mode, m):
    """The derivative through the host streaming path (row chunks and segment
    chunks) and the range entry: the halo geometry t0 = M, L = N - M - 1
    (ols.py:137-146); for M = 1 too (where the reference recomputes seam
    neighbours from the input).  Streaming is bit-identical to the device
    path; all of it agrees with the float64 direct convolution's global
    difference within the fp32 bar, and the Executor matches convolve()."""
    from paper_1910_01972_b200.ols import fused_range_launch
    ns, nfil, n, origin = 20001, 3, 256, (m // 2)
    rng = np.random.default_rng([93, ns, m])
    real = mode == "r2r"
    x = rng.standard_normal(ns) if real else (rng.standard_normal(ns)
                                              + 1j * rng.standard_normal(ns))
    taps = rng.standard_normal((nfil, m)) if real else (
        rng.standard_normal((nfil, m)) + 1j * rng.standard_normal((nfil, m)))
    P = oc.Precision.single
    vk = "real" if real else "complex"
    p = oc.plan(ns, m, mode, origin, n)
    pp = oc.PostProcSpec("derivative")
    fs = oc.transform_filters(oc.make_filterset(taps, origin, P), p,
                              "natural" if real else "permuted")
    sig = oc.make_signal(x, vk, P)
    dev = oc.convolve(sig, fs, p, postproc=pp)
    # reference: global central difference of the float64 convolution
    import oracle
    y = oracle.direct_convolve(x, taps, origin)
    y = y.real if real else y
    d = np.empty_like(y)
    d[:, 1:-1] = 0.5 * (y[:, 2:] - y[:, :-2])
    d[:, 0] = y[:, 1] - y[:, 0]
    d[:, -1] = y[:, -1] - y[:, -2]
    assert rel_l2_per_filter(dev.cpu().numpy(), d) <= 2 * L2_TOL
    hsig = oc.make_signal(torch.from_numpy(np.ascontiguousarray(x).astype(
        np.float32 if real else np.complex64)).pin_memory(), vk, P, device="cpu")
    for chunk in (None, 7):
        host = torch.full(tuple(dev.shape), float("nan"),
                          dtype=dev.dtype).pin_memory()
        oc.convolve(hsig, fs, p, postproc=pp, out=host, chunk_segments=chunk)
        assert torch.equal(host, dev.cpu()), chunk
    # a range launch in the middle of the signal
    lo, hi = 6000, 13001
    out = torch.empty((nfil, hi - lo), dtype=dev.dtype, device="cuda")
    fused_range_launch(sig.samples, 0, ns, fs.spectra_dev, nfil, p, lo, hi, pp,
                       out, hi - lo, lo, P)
    assert torch.equal(out, dev[:, lo:hi])
    ex = oc.Executor(fs, p, pp)
    assert torch.equal(ex(sig), dev)
