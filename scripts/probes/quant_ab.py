"""A/B of kvq_quantize (a3 alone) geometries at C4: KVQ_QSLAB_U = 0 (persistent) / 4 / 8 / 16, bit-identical check."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2601_04719_b200 import kvq  # noqa: E402

T, D = 131072, 8192
K = kvq.kvq_synth_fill(T, D, seed=42)
s = kvq.kvq_compute_scales(K)
q = torch.empty(T, D, dtype=torch.int8, device="cuda")
st = torch.cuda.current_stream()


def t(n=20):
    for _ in range(3):
        kvq.kvq_quantize(K, s, q, stream=st)
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kvq.kvq_compute_scales(K, s, stream=st)  # what precedes it in the separate pipeline
        a.record(st)
        kvq.kvq_quantize(K, s, q, stream=st)
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return round(statistics.median(ts), 4)


os.environ["KVQ_QSLAB_U"] = "0"
t(3)
ref = q.clone()
for rep in range(2):
    for u in ("0", "4", "8", "16"):
        os.environ["KVQ_QSLAB_U"] = u
        ms = t()
        print(f"U={u} quantize C4 {ms} ms  {5 * T * D / ms / 1e6:.0f} GB/s  identical={torch.equal(q, ref)}", flush=True)
