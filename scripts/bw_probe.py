"""Characterise B200 HBM for this path's traffic mix with plain torch ops (no kvq code):
read-only (amax over 4.3 GB), write-only (fill_ of 4.3 GB), copy (1:1).  Median of 20."""
import json
import statistics

import torch

N = 1 << 30
x = torch.empty(N, dtype=torch.float32, device="cuda").uniform_()
y = torch.empty(N, dtype=torch.float32, device="cuda")


def t(fn, iters=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


res = {}
ms = t(lambda: torch.amax(x))
res["read_only_GBps"] = 4 * N / (ms * 1e-3) / 1e9
ms = t(lambda: y.fill_(1.0))
res["write_only_GBps"] = 4 * N / (ms * 1e-3) / 1e9
ms = t(lambda: y.copy_(x))
res["copy_1to1_GBps"] = 8 * N / (ms * 1e-3) / 1e9
print(json.dumps(res))

# write-heavy (1 B read : 4 B write) and read-heavy (4 B : 1 B) conversions, torch kernels
q8 = torch.randint(-127, 128, (N,), dtype=torch.int8, device="cuda")
ms = t(lambda: y.copy_(q8))
res["int8_to_f32_GBps(1R:4W)"] = 5 * N / (ms * 1e-3) / 1e9
ms = t(lambda: q8.copy_(x))
res["f32_to_int8_GBps(4R:1W)"] = 5 * N / (ms * 1e-3) / 1e9
z = torch.empty(N, dtype=torch.float32, device="cuda")
ms = t(lambda: torch.add(x, x, out=z))
res["add_1R1W_GBps"] = 8 * N / (ms * 1e-3) / 1e9
print(json.dumps(res))
