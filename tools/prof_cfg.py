"""Run one BASELINE config through the fused engine a few times (for ncu).

    python tools/prof_cfg.py cfg3 [reps]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import paper_1910_01972_b200 as ob  # noqa: E402
from cases import gen_inputs  # noqa: E402

CFG = {
    "cfg1": (1 << 20, 64, 1, 1024),
    "cfg3": (1 << 23, 400, 96, 2048),
    "cfg2_n256": (1 << 22, 64, 32, 256),
    "cfg2_n512": (1 << 22, 128, 32, 512),
    "cfg2_n1024": (1 << 22, 256, 32, 1024),
    "cfg2_n2048": (1 << 22, 512, 32, 2048),
    "cfg2_n4096": (1 << 22, 1024, 32, 4096),
    "cfg4_m8_f8": (1 << 24, 8, 8, 64),
    "cfg4_m32_f8": (1 << 24, 32, 8, 128),
    "cfg4_m8_f1": (1 << 24, 8, 1, 64),
    "cfg4_m16_f1": (1 << 24, 16, 1, 64),
    "cfg4_m32_f1": (1 << 24, 32, 1, 128),
    "cfg4_m16_f8": (1 << 24, 16, 8, 64),
    "cfg4_m8_f4": (1 << 24, 8, 4, 64),
    "cfg4_m8_f2": (1 << 24, 8, 2, 64),
    "cfg1_f2": (1 << 20, 64, 2, 1024),
    "cfg1_f4": (1 << 20, 64, 4, 1024),
    # cfg5's per-GPU share at 8 GPUs (2^30 / 8 samples, 64 filters M=512)
    "cfg5_shard8": (1 << 27, 512, 64, 4096),
    # real (r2r) path on the same shapes
    "cfg3_r2r": (1 << 23, 400, 96, 2048, "r2r"),
    "cfg2_n1024_r2r": (1 << 22, 256, 32, 1024, "r2r"),
    "cfg2_n4096_r2r": (1 << 22, 1024, 32, 4096, "r2r"),
}

if __name__ == "__main__":
    name = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    ns, m, nfil, n, *mode = CFG[name]
    mode = mode[0] if mode else "c2c"
    x, taps = gen_inputs(ns, m, nfil)
    P = ob.Precision.single
    if mode == "r2r":
        x, taps = x.real, taps.real
    sig = ob.make_signal(x, "real" if mode == "r2r" else "complex", P)
    p = ob.plan(ns, m, mode, 0, n)
    fs = ob.transform_filters(ob.make_filterset(taps, 0, P), p,
                              "natural" if mode == "r2r" else "permuted")
    out = torch.empty((nfil, ns), dtype=torch.float32 if mode == "r2r"
                      else torch.complex64, device="cuda")
    for _ in range(reps):
        ob.convolve(sig, fs, p, out=out)
    torch.cuda.synchronize()
    print("done", name)
