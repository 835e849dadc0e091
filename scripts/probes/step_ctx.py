"""In-step timing of the headline step's two passes (colmax, roundtrip) under different contexts:
roundtrip tile order (KVQ_TC_HINTS bit 2 = last tile first), an L2 flush between the passes.

    python scripts/probes/step_ctx.py
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2601_04719_b200 import kvq  # noqa: E402

T, D, nq = 131072, 8192, 64
K = kvq.kvq_synth_fill(T, D, seed=42)
Q = kvq.kvq_synth_fill(nq, D, seed=43)
s = kvq.kvq_compute_scales(K)
Kq = torch.empty(T, D, dtype=torch.int8, device="cuda")
Kh = torch.empty(T, D, dtype=torch.float32, device="cuda")
ws = torch.empty(kvq.kvq_roundtrip_workspace_size(T, D, nq), dtype=torch.uint8, device="cuda")
mout = torch.empty(kvq.METRICS_BYTES, dtype=torch.uint8, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()


def run(n=30, flush_between=False):
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n)]
    for i in range(n + 5):
        e = ev[i - 5] if i >= 5 else None
        if e: e[0].record(st)
        kvq.kvq_compute_scales(K, s, stream=st)
        if e: e[1].record(st)
        if flush_between:
            flush.fill_(1.0)
            if e: e[1].record(st)
        kvq.kvq_roundtrip(K, s, Q, Kq, Kh, out_dev=mout, workspace=ws, stream=st)
        if e: e[2].record(st)
    torch.cuda.synchronize()
    c = statistics.median(a.elapsed_time(b) for a, b, _ in ev)
    r = statistics.median(b.elapsed_time(x) for _, b, x in ev)
    return round(c, 4), round(r, 4)


print(os.environ.get("KVQ_TC_HINTS", "3"), "step (colmax, roundtrip) ms:", run(), flush=True)
print(os.environ.get("KVQ_TC_HINTS", "3"), "with 256 MB flush before the roundtrip:", run(flush_between=True), flush=True)
