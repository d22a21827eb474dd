"""Per-call overhead of convolve() on small cells (launch-bound regime).

    python tools/overhead.py
Prints host wall time per call (back-to-back calls, one sync at the end),
device time per call (CUDA events around a batch) and the kernel time from a
CUDA-graph replay of the raw C-ABI launch.
"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import paper_1910_01972_b200 as ob  # noqa: E402
from paper_1910_01972_b200.ols import _geometry, fused_launch  # noqa: E402
from cases import gen_inputs  # noqa: E402

for ns, m, nfil, n in [(1 << 20, 64, 1, 1024), (1 << 16, 64, 4, 256)]:
    x, taps = gen_inputs(ns, m, nfil)
    P = ob.Precision.single
    sig = ob.make_signal(x, "complex", P)
    p = ob.plan(ns, m, "c2c", 0, n)
    fs = ob.transform_filters(ob.make_filterset(taps, 0, P), p, "permuted")
    out = torch.empty((nfil, ns), dtype=torch.complex64, device="cuda")
    for _ in range(20):
        ob.convolve(sig, fs, p, out=out)
    torch.cuda.synchronize()
    reps = 500
    t0 = time.perf_counter()
    for _ in range(reps):
        ob.convolve(sig, fs, p, out=out)
    torch.cuda.synchronize()
    host_us = (time.perf_counter() - t0) / reps * 1e6
    # raw launch captured in a CUDA graph: device time of the kernel alone
    l_eff, t0g, win_off, n_seg = _geometry(p, 0)
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        fused_launch(sig.samples, 0, ns, fs.spectra_dev, nfil, p, l_eff, t0g,
                     win_off, 0, n_seg, ob.NONE, out, ns, 0, P)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            for _ in range(20):
                fused_launch(sig.samples, 0, ns, fs.spectra_dev, nfil, p, l_eff,
                             t0g, win_off, 0, n_seg, ob.NONE, out, ns, 0, P)
    g.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    e1.synchronize()
    graph_us = e0.elapsed_time(e1) / 20 * 1e3
    ex = ob.Executor(fs, p)
    for _ in range(20):
        ex(sig, out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        ex(sig, out)
    torch.cuda.synchronize()
    ex_us = (time.perf_counter() - t0) / reps * 1e6
    print(f"ns={ns} m={m} F={nfil} N={n}: convolve() host {host_us:.1f} us/call, "
          f"Executor host {ex_us:.1f} us/call, "
          f"graph-replayed kernel {graph_us:.1f} us, traffic at HBM peak "
          f"{8 * ns * (1 + nfil) / 6.546e12 * 1e6:.1f} us", flush=True)
