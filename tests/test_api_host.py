"""Host-side API parity with the reference (no GPU needed).

Planner arithmetic, validation order and exceptions mirror
olsconv/ols.py:53-155 and fft.py:85-99; cases are the reference's own
(tests/test_ols.py:15-75, test_fft.py:66-95).
"""

import numpy as np
import pytest

import paper_1910_01972_b200 as oc
from paper_1910_01972_b200 import PostProcSpec
from paper_1910_01972_b200.ols import _chunk_bounds, _geometry


def test_plan_sweep_point():
    p = oc.plan(2_000_000, 1025, "c2c", 0, 4096)
    assert p.valid_len == 3072 and p.n_segments == 652


def test_plan_degenerate_single_tap():
    p = oc.plan(10, 1, "c2c", 0, 4)
    assert p.valid_len == 4 and p.n_segments == 3


def test_plan_errors():
    with pytest.raises(oc.SegmentTooSmall):
        oc.plan(100, 64, "c2c", 0, 32)
    with pytest.raises(oc.FilterTooLong):
        oc.plan(1000, 5000, "c2c")
    with pytest.raises(oc.BadLength):
        oc.plan(100, 3, "c2c", 0, 100)
    with pytest.raises(oc.BadLength):
        oc.plan(100, 3, "r2r", 0, 4)
    with pytest.raises(ValueError):
        oc.plan(100, 3, "xyz")
    with pytest.raises(ValueError):
        oc.plan(0, 3, "c2c")
    with pytest.raises(ValueError):
        oc.plan(100, 3, "c2c", origin=3)


def test_plan_auto_defaults():
    assert oc.plan(1000, 1, "c2c").fft_len == 64
    assert oc.plan(1000, 129, "c2c").fft_len == 512
    assert oc.plan(1000, 4000, "c2c").fft_len == 4096
    assert oc.auto_segment_len(65, "pipelined") == 8192
    # cfg4 auto lengths (SURVEY §8 geometry table)
    assert [oc.plan(1 << 24, m, "c2c").fft_len for m in (8, 16, 32)] == \
        [64, 64, 128]


def test_plan_invariants_over_grid():
    for n_s in (1, 10, 1000, 12345):
        for m in (1, 3, 17, 64):
            for n in (64, 256):
                p = oc.plan(n_s, m, "c2c", 0, n)
                assert p.valid_len == n - m + 1 >= 1
                assert p.n_segments * p.valid_len >= n_s
                assert (p.n_segments - 1) * p.valid_len < n_s


def test_baseline_geometry_table():
    # L and n_seg per config
    rows = [((1 << 20, 64, 1024), (961, 1092)),
            ((1 << 22, 64, 256), (193, 21733)),
            ((1 << 22, 1024, 4096), (3073, 1365)),
            ((1 << 23, 400, 2048), (1649, 5088)),
            ((1 << 30, 512, 4096), (3585, 299510))]
    for (ns, m, n), (l, nseg) in rows:
        p = oc.plan(ns, m, "c2c", 0, n)
        assert (p.valid_len, p.n_segments) == (l, nseg)


def test_output_windows_partition():
    for n_s in (1, 7, 1000, 4097):
        for m, n in ((1, 64), (17, 64), (62, 64), (129, 1024)):
            for pp in (oc.NONE, PostProcSpec("derivative")):
                p = oc.plan(n_s, m, "c2c", 0, n)
                counts = np.zeros(n_s, dtype=int)
                for lo, hi in oc.output_windows(p, pp):
                    assert 0 <= lo < hi <= n_s
                    counts[lo:hi] += 1
                assert np.all(counts == 1)


def test_output_windows_halo_infeasible():
    p = oc.plan(1000, 63, "c2c", 0, 64)
    with pytest.raises(oc.HaloUnavailable):
        oc.output_windows(p, PostProcSpec("derivative"))


def test_geometry_no_halo():
    p = oc.plan(5000, 33, "c2c", 16, 128)
    assert _geometry(p, 0) == (96, 32, 16 - 32, -(-5000 // 96))


def test_chunk_bounds_is_reference_split():
    assert _chunk_bounds(10, 3) == [(0, 4), (4, 8), (8, 10)]
    assert _chunk_bounds(2, 8) == [(0, 1), (1, 2)]
    assert _chunk_bounds(5088, 1) == [(0, 5088)]


def test_make_plan_validation():
    p = oc.make_plan(4096, "ct_dif_permuted")
    assert p.length == 4096 and p.twiddles.shape == (2048,)
    assert p.layout == "bit_reversed"
    with pytest.raises(oc.BadLength):
        oc.make_plan(3000, "stockham")
    with pytest.raises(oc.BadLength):
        oc.make_plan(8192, "stockham")
    oc.make_plan(8192, "stockham", max_len=8192)
    with pytest.raises(oc.BadLength):
        oc.make_plan(4, "real_packed")
    with pytest.raises(ValueError):
        oc.make_plan(64, "radix3")


def test_twiddles_match_reference_tables():
    import oracle
    for n in (4, 64, 2048):
        p = oc.make_plan(n, "ct_dif_permuted")
        tw, twc = oracle.tables(n, "single")
        assert np.array_equal(p.twiddles, tw)
        assert np.array_equal(p.twiddles_conj, twc)


def test_bit_reverse_and_naive_dft():
    assert oc.bit_reverse_permutation(1, 3) == 4
    assert oc.bit_reverse_permutation(6, 4) == 6
    with pytest.raises(ValueError):
        oc.bit_reverse_permutation(8, 3)
    assert np.allclose(oc.naive_dft([1, 1]), [2, 0])
    assert np.allclose(oc.naive_dft(oc.naive_dft([1, 2, 3]), "inverse"),
                       [1, 2, 3])


def test_postproc_spec():
    assert PostProcSpec().code == 0 and PostProcSpec("scale", 2).code == 1
    assert PostProcSpec("derivative").halo == 1
    assert PostProcSpec("magnitude_squared").real_output
    with pytest.raises(ValueError):
        PostProcSpec("cube")


def test_error_hierarchy_matches_reference():
    names = ["EmptyInput", "RaggedFilters", "BadOrigin", "DomainMismatch",
             "BadLength", "BadSpectrum", "FilterTooLong", "SegmentTooSmall",
             "PlanMismatch", "LayoutMismatch", "HaloUnavailable", "TooLarge"]
    for n in names:
        assert issubclass(getattr(oc, n), oc.OlsError)
    assert issubclass(oc.EngineError, RuntimeError)


def test_public_names_cover_reference_api():
    # every name of olsconv.__all__ (olsconv/__init__.py:22-39) except the
    # oracle entry points (test infrastructure here) and apply_postproc
    ref_names = [
        "BACKEND", "backend_name", "CONV_TOL", "FFT_TOL", "FilterSet",
        "Precision", "Signal", "make_filterset", "make_signal", "BadLength",
        "BadOrigin", "BadSpectrum", "DomainMismatch", "EmptyInput",
        "FilterTooLong", "HaloUnavailable", "LayoutMismatch", "OlsError",
        "PlanMismatch", "RaggedFilters", "SegmentTooSmall", "TooLarge",
        "DEFAULT_MAX_FFT_LEN", "FftPlan", "bit_reverse_permutation",
        "fft_forward_permuted", "fft_inverse_permuted", "fft_stockham",
        "irfft_packed", "make_plan", "naive_dft", "rfft_packed",
        "ENGINE_VARIANTS", "MODES", "SegmentPlan", "auto_segment_len",
        "autotune_segment_size", "convolve", "full_fft_convolve",
        "measure_segment_times", "output_windows", "plan",
        "transform_filters", "NONE", "PostProcSpec", "__version__"]
    for n in ref_names:
        assert hasattr(oc, n), n
