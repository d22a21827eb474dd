"""Sustained-run probe: back-to-back fused launches on one config while
nvidia-smi samples SM clock, power draw and throttle reasons (20 ms).

    python tools/power_probe.py cfg3 [seconds]
Prints per-window kernel time (CUDA events over 10 launches) with the clock
and power samples that fell inside the window.
"""
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden"),
                os.path.join(ROOT, "tools")]

import paper_1910_01972_b200 as ob  # noqa: E402
from cases import gen_inputs  # noqa: E402
from prof_cfg import CFG  # noqa: E402


def main():
    name = sys.argv[1]
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
    ns, m, nfil, n, *_ = CFG[name]
    x, taps = gen_inputs(ns, m, nfil)
    P = ob.Precision.single
    sig = ob.make_signal(x, "complex", P)
    p = ob.plan(ns, m, "c2c", 0, n)
    fs = ob.transform_filters(ob.make_filterset(taps, 0, P), p, "permuted")
    out = torch.empty((nfil, ns), dtype=torch.complex64, device="cuda")
    ex = ob.Executor(fs, p)
    ex(sig.samples, out)
    torch.cuda.synchronize()
    samples = []
    proc = subprocess.Popen(
        ["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,"
         "clocks_event_reasons.sw_power_cap,temperature.gpu",
         "--format=csv,noheader,nounits", "-lms", "20"],
        stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

    def rd():
        for ln in proc.stdout:
            samples.append((time.time(), ln.strip()))
    th = threading.Thread(target=rd, daemon=True)
    th.start()
    time.sleep(0.3)
    t_end = time.time() + secs
    wins = []
    while time.time() < t_end:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        w0 = time.time()
        e0.record()
        for _ in range(10):
            ex(sig.samples, out)
        e1.record()
        e1.synchronize()
        wins.append((w0, time.time(), e0.elapsed_time(e1) / 10))
    time.sleep(0.2)
    proc.terminate()
    for w0, w1, ms in wins[:: max(1, len(wins) // 12)]:
        sm = [s.split(",") for t, s in samples if w0 <= t <= w1]
        clk = np.median([float(v[0]) for v in sm]) if sm else float("nan")
        pw = np.median([float(v[1]) for v in sm]) if sm else float("nan")
        cap = sum("Active" in v[2] for v in sm)
        tmp = sm[-1][3].strip() if sm else "?"
        print(f"{name} t+{w0 - wins[0][0]:5.2f}s  {ms:.3f} ms/launch  "
              f"sm {clk:.0f} MHz  {pw:.0f} W  power_cap {cap}/{len(sm)}  "
              f"{tmp} C", flush=True)


if __name__ == "__main__":
    main()
