"""Event-timed kvq_roundtrip / quantize / dequantize / colmax at C4 (or T D from argv), for A/B experiments.

    python scripts/time_rt.py [T] [D]          (KVQ_TC_HINTS etc. are read by the library)
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_04719_b200 import kvq  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
D = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
nq = 64
K = kvq.kvq_synth_fill(T, D, seed=42)
Q = kvq.kvq_synth_fill(nq, D, seed=43)
s = kvq.kvq_compute_scales(K)
Kq = torch.empty(T, D, dtype=torch.int8, device="cuda")
Kh = torch.empty(T, D, dtype=torch.float32, device="cuda")
ws = torch.empty(kvq.kvq_roundtrip_workspace_size(T, D, nq), dtype=torch.uint8, device="cuda")
mout = torch.empty(kvq.METRICS_BYTES, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def t(fn, n=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return round(statistics.median(ts), 4), round(min(ts), 4)


res = {
    "roundtrip": t(lambda: kvq.kvq_roundtrip(K, s, Q, Kq, Kh, out_dev=mout, workspace=ws, stream=st)),
    "scales": t(lambda: kvq.kvq_compute_scales(K, s, stream=st)),
    "quantize": t(lambda: kvq.kvq_quantize(K, s, Kq, stream=st)),
    "dequantize": t(lambda: kvq.kvq_dequantize(Kq, s, Kh, stream=st)),
    "quant+dequant": t(lambda: kvq.kvq_quantize_dequantize(K, s, Kq, Kh, stream=st)),
}
print(os.environ.get("KVQ_TC_HINTS", "-"), T, D, res, flush=True)
