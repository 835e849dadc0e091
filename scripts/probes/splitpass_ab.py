"""A/B: kvq_roundtrip as one tile pass (K_hat + codes in tile order) vs a codes-only tile pass + a linear
row-slab dequantize (KVQ_RT_SPLITPASS=1).  In-step timing, outputs checked identical."""
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
st = torch.cuda.current_stream()


def run(n=30):
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n)]
    for i in range(n + 5):
        e = ev[i - 5] if i >= 5 else None
        if e: e[0].record(st)
        kvq.kvq_compute_scales(K, s, stream=st)
        if e: e[1].record(st)
        kvq.kvq_roundtrip(K, s, Q, Kq, Kh, out_dev=mout, workspace=ws, stream=st)
        if e: e[2].record(st)
    torch.cuda.synchronize()
    return (round(statistics.median(a.elapsed_time(b) for a, b, _ in ev), 4),
            round(statistics.median(b.elapsed_time(x) for _, b, x in ev), 4))


os.environ["KVQ_RT_SPLITPASS"] = "0"
run(3)
ref = (Kq.clone(), Kh.clone(), mout.clone())
for rep in range(3):
    for v in ("0", "1"):
        os.environ["KVQ_RT_SPLITPASS"] = v
        Kq.zero_(); Kh.zero_()
        t = run()
        same = all(torch.equal(a, b) for a, b in zip(ref, (Kq, Kh, mout)))
        print(f"splitpass={v} (colmax, roundtrip) ms {t} identical={same}", flush=True)
