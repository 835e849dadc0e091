"""Event-timed kvq_error_metrics_async (a5+a6, tensor-core kernel MODE 0) at C4."""
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
Kh = kvq.kvq_dequantize(kvq.kvq_quantize(K, s), s)
ws = torch.empty(kvq.kvq_error_metrics_workspace_size(T, D, nq), dtype=torch.uint8, device="cuda")
mout = torch.empty(kvq.METRICS_BYTES, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
ts = []
for i in range(25):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    kvq.kvq_error_metrics_async(K, Kh, Q, s, out_dev=mout, workspace=ws, stream=st)
    b.record(st)
    b.synchronize()
    if i >= 5:
        ts.append(a.elapsed_time(b))
print("metrics C4 ms median", round(statistics.median(ts), 4), "min", round(min(ts), 4),
      "GB/s (8 B/elem, median)", round(8 * T * D / statistics.median(ts) / 1e6, 1), flush=True)
