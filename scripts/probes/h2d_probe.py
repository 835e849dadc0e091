"""Raw pinned host<->device copy bandwidth (the e2e path's ceiling): 4.3 GB H2D, 1.07 GB D2H, and both at once."""
import time
import torch

n = 131072 * 8192
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
hc = torch.empty(n, dtype=torch.int8).pin_memory()
dc = torch.empty(n, dtype=torch.int8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
h2d = 3 * n * 4 / (time.perf_counter() - t) / 1e9
t = time.perf_counter()
for _ in range(3):
    hc.copy_(dc, non_blocking=True)
torch.cuda.synchronize()
d2h = 3 * n / (time.perf_counter() - t) / 1e9
t = time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        hc.copy_(dc, non_blocking=True)
torch.cuda.synchronize()
both = time.perf_counter() - t
print({"h2d_GBps": h2d, "d2h_GBps": d2h, "duplex_h2d_GBps": 3 * n * 4 / both / 1e9})
