import torch, time
d = torch.empty(1<<30, dtype=torch.uint8, device='cuda')
h = torch.empty(1<<30, dtype=torch.uint8).pin_memory()
for chunk in (16<<20, 64<<20, 256<<20, 1<<30):
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(3):
        for o in range(0, 1<<30, chunk):
            h[o:o+chunk].copy_(d[o:o+chunk], non_blocking=True)
    e1.record(); e1.synchronize()
    print(f"D2H chunk {chunk>>20} MiB: {3*(1<<30)/e0.elapsed_time(e1)/1e6:.1f} GB/s")
# two streams
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
torch.cuda.synchronize(); t=time.time()
for r in range(3):
    with torch.cuda.stream(s1): h[:1<<29].copy_(d[:1<<29], non_blocking=True)
    with torch.cuda.stream(s2): h[1<<29:].copy_(d[1<<29:], non_blocking=True)
torch.cuda.synchronize(); print(f"D2H 2 streams: {3*(1<<30)/(time.time()-t)/1e9:.1f} GB/s")
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record()
for r in range(3): d.copy_(h, non_blocking=True)
e1.record(); e1.synchronize(); print(f"H2D: {3*(1<<30)/e0.elapsed_time(e1)/1e6:.1f} GB/s")
