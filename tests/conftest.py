"""Shared test helpers (mirrors the reference's tests/conftest.py:6-38).

Markers: ``gpu`` = needs a CUDA device (run on the B200 box with -m gpu);
everything else runs on the CPU-only build container.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def rel_err(got, ref):
    """Relative L-inf error, the reference's acceptance metric
    (tests/conftest.py:6-10)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    scale = float(np.abs(ref).max()) or 1.0
    return float(np.abs(got - ref).max()) / scale


def rel_l2_per_filter(got, ref):
    """max over filters of ||got_f - ref_f||_2 / ||ref_f||_2 — the
    north_star parity metric (tolerance 1e-5 for fp32)."""
    got = np.atleast_2d(np.asarray(got))
    ref = np.atleast_2d(np.asarray(ref))
    num = np.sqrt(np.sum(np.abs(got.astype(np.complex128) - ref) ** 2, axis=-1))
    den = np.sqrt(np.sum(np.abs(ref) ** 2, axis=-1))
    return float(np.max(num / np.maximum(den, 1e-300)))


def rng_for(*key):
    return np.random.default_rng(list(key))


@pytest.fixture(scope="session")
def golden():
    return {
        "fft": np.load(os.path.join(GOLDEN, "fft_permuted.npz")),
        "spectra": np.load(os.path.join(GOLDEN, "spectra.npz")),
        "conv": np.load(os.path.join(GOLDEN, "conv_cases.npz")),
        "cfg": np.load(os.path.join(GOLDEN, "cfg_windows.npz")),
        "pp": np.load(os.path.join(GOLDEN, "pp_cases.npz")),
    }


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
