"""Device->pinned-host copy bandwidth: one 2 GiB copy, 64 MiB chunks, and two streams."""
import time

import torch

dev = torch.device("cuda", 0)
nb = 2 << 30
src = torch.empty(nb // 8, dtype=torch.float64, device=dev).fill_(1.0)
dst = torch.empty(nb // 8, dtype=torch.float64).pin_memory()
dst2 = torch.empty(nb // 8, dtype=torch.float64).pin_memory()
for name, chunk in (("single", nb), ("64MiB", 64 << 20), ("8MiB", 8 << 20)):
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        e = chunk // 8
        for o in range(0, nb // 8, e):
            dst[o:o + e].copy_(src[o:o + e], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"D2H {name}: {nb / dt / 1e9:.1f} GB/s")
torch.cuda.synchronize()
t = time.perf_counter()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h = nb // 16
with torch.cuda.stream(s1):
    dst[:h].copy_(src[:h], non_blocking=True)
with torch.cuda.stream(s2):
    dst[h:].copy_(src[h:], non_blocking=True)
torch.cuda.synchronize()
print(f"D2H two streams: {nb / (time.perf_counter() - t) / 1e9:.1f} GB/s")
t = time.perf_counter()
hsrc = dst2
d2 = torch.empty_like(src)
d2.copy_(hsrc, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D single: {nb / (time.perf_counter() - t) / 1e9:.1f} GB/s")
