"""The experimental fused engines selected by environment switches (DESIGN.md
§5.4): the warp-per-segment N = 2048 engine (OLSB_W64=1), the two-warp N =
4096 engine (OLSB_W64X2=1) and the two-warp E = 32 N = 2048 engine
(OLSB_W32X2=1).  The switches are read once per process, so each runs in a
subprocess; every engine is checked against the reference's float64 golden
outputs (fp32 bar) on cells that exercise its N, first / last segments,
origin > 0, partial output ranges and |y|^2."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path[:0] = [%(root)r, %(root)r + "/tests", %(root)r + "/tests/golden"]
import oracle
import paper_1910_01972_b200 as oc
from paper_1910_01972_b200.ols import fused_range_launch
from conftest import rel_l2_per_filter
worst = 0.0
for (ns, m, nfil, n, origin) in %(cells)r:
    rng = np.random.default_rng([123, ns, m, n])
    x = rng.standard_normal(ns) + 1j * rng.standard_normal(ns)
    taps = rng.standard_normal((nfil, m)) + 1j * rng.standard_normal((nfil, m))
    P = oc.Precision.single
    p = oc.plan(ns, m, "c2c", origin, n)
    fs = oc.transform_filters(oc.make_filterset(taps, origin, P), p, "permuted")
    sig = oc.make_signal(x, "complex", P)
    ref = oracle.direct_convolve(x, taps, origin)
    y = oc.convolve(sig, fs, p).cpu().numpy()
    worst = max(worst, rel_l2_per_filter(y, ref))
    a2 = oc.convolve(sig, fs, p, postproc=oc.PostProcSpec("magnitude_squared"))
    worst = max(worst, rel_l2_per_filter(a2.cpu().numpy(), np.abs(ref) ** 2) / 2)
    lo, hi = ns // 3 + 7, 2 * ns // 3 + 1
    out = torch.full((nfil, hi - lo), float("nan"), dtype=torch.complex64,
                     device="cuda")
    fused_range_launch(sig.samples, 0, ns, fs.spectra_dev, nfil, p, lo, hi,
                       oc.NONE, out, hi - lo, lo, P)
    worst = max(worst, rel_l2_per_filter(out.cpu().numpy(), ref[:, lo:hi]))
print("WORST", worst)
'''


@pytest.mark.parametrize("env,n", [("OLSB_W64", 2048), ("OLSB_W32X2", 2048),
                                   ("OLSB_W64X2", 4096)])
def test_experimental_engine_parity(env, n):
    m = n // 4 + 17
    cells = [(3 * n + 5, m, 3, n, 0), (20 * n + 11, m, 5, n, m // 3),
             (n // 2, m, 2, n, 1)]
    code = SCRIPT % {"root": ROOT, "cells": cells}
    res = subprocess.run([sys.executable, "-c", code], capture_output=True,
                         text=True, env=dict(os.environ, **{env: "1"}),
                         timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    worst = float(res.stdout.split("WORST")[-1])
    assert worst <= 1e-5, (env, worst)


@pytest.mark.parametrize("val", ["1", "2", "3"])
def test_tma_spectrum_ring_parity(val):
    """OLSB_HTMA: filter spectra through the shared-memory TMA ring (full /
    empty mbarriers, one filter ahead) -- 1: TMEM residency, 2: TMX = 1,
    3: register policy; F = 1 cells take the register policy.  Filter counts
    1-5 exercise the ring's slot and phase turnover across items."""
    cells = []
    for n in (64, 256, 1024, 2048, 4096):
        m = n // 4 + 1
        cells += [(3 * n + 5, m, 1, n, 0), (20 * n + 11, m, 5, n, m // 3),
                  (9 * n + 3, m, 2, n, 1)]
    code = SCRIPT % {"root": ROOT, "cells": cells}
    res = subprocess.run([sys.executable, "-c", code], capture_output=True,
                         text=True, env=dict(os.environ, OLSB_HTMA=val),
                         timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    worst = float(res.stdout.split("WORST")[-1])
    assert worst <= 1e-5, (val, worst)
