"""Graph-replay floor of a cfg1-sized cell: what a plain device copy with
cfg1's traffic (read 8 MiB + write 8 MiB per filter) and a trivial kernel
take per launch when replayed back to back, next to the engine's cfg1 time
(tools/time_graph.py)."""
import torch


def per_launch(fn, n=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    ts = []
    for _ in range(6):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / n)
    ts.sort()
    return ts[len(ts) // 2] * 1e3


ns = 1 << 20
for nfil in (1, 2):
    src = torch.randn(ns, dtype=torch.complex64, device="cuda")
    dst = torch.empty((nfil, ns), dtype=torch.complex64, device="cuda")
    t = per_launch(lambda: dst.copy_(src.expand(nfil, ns)))
    print(f"copy 8 MiB -> {nfil} x 8 MiB (cfg1{'_f2' if nfil == 2 else ''} traffic): "
          f"{t:.1f} us per launch", flush=True)
tiny = torch.zeros(32, device="cuda")
print(f"trivial kernel: {per_launch(lambda: tiny.add_(1)):.1f} us per launch")
