"""H2D bandwidth from pinned host memory with 1, 2 and 4 concurrent copy
streams (frames interleaved over the streams), and SM-driven reads of host
memory alongside (the question: is one copy engine the limit, or PCIe?)."""
import time

import torch

n = 4 << 30
frame = 128 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(k)]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, off in enumerate(range(0, n, frame)):
            with torch.cuda.stream(ss[i % k]):
                d[off:off + frame].copy_(h[off:off + frame], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"streams {k}: h2d {n / dt / 1e9:.1f} GB/s", flush=True)
# both directions at once
torch.cuda.synchronize()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"h2d+d2h concurrently: {2 * n / (time.perf_counter() - t0) / 1e9:.1f} GB/s total", flush=True)
