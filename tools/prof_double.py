import os, sys
import torch
ROOT = "/root/repo" if os.path.exists("/root/repo") else os.getcwd()
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden")]
import paper_1910_01972_b200 as ob
from cases import gen_inputs
ns, m, nfil, n = 1 << 23, 400, 96, 2048
x, taps = gen_inputs(ns, m, nfil)
P = ob.Precision.double
sig = ob.make_signal(x, "complex", P)
p = ob.plan(ns, m, "c2c", 0, n)
fs = ob.transform_filters(ob.make_filterset(taps, 0, P), p, "permuted")
out = torch.empty((nfil, ns), dtype=torch.complex128, device="cuda")
for _ in range(2):
    ob.convolve(sig, fs, p, out=out)
torch.cuda.synchronize()
