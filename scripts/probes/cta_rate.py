"""Per-CTA rate of the fused tensor-core roundtrip (attn_tc_kernel<2>) vs the number of tiles in flight:
whole 128-row tiles, D = 8192 (256 K-blocks per tile), one wave of `tiles` CTAs.  If the time per K-block
stays flat from 8 to 148 CTAs (and with L2-resident inputs), the pass is bound per CTA, not by HBM.

    KVQ_TC_BALANCE=0 python scripts/probes/cta_rate.py
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2601_04719_b200 import kvq  # noqa: E402

D, nq = int(os.environ.get("D", 8192)), 64
st = torch.cuda.current_stream()
Q = kvq.kvq_synth_fill(nq, D, seed=43)
for tiles in [int(x) for x in os.environ.get("TILES", "8,16,32,64,96,128,148,296,592").split(",")]:
    T = tiles * 128
    K = kvq.kvq_synth_fill(T, D, seed=42)
    s = kvq.kvq_compute_scales(K)
    Kq = torch.empty((T, D), dtype=torch.int8, device="cuda")
    Kh = torch.empty((T, D), dtype=torch.float32, device="cuda")
    ws = torch.empty(kvq.kvq_roundtrip_workspace_size(T, D, nq), dtype=torch.uint8, device="cuda")
    mout = torch.empty(kvq.METRICS_BYTES, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(25):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        torch.cuda._sleep(50000)
        a.record(st)
        kvq.kvq_roundtrip(K, s, Q, Kq, Kh, out_dev=mout, workspace=ws, stream=st)
        b.record(st)
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    waves = -(-tiles // 148)
    kb = waves * ((D + 31) // 32)
    gbs = 9 * T * D / (ms * 1e-3) / 1e9
    print(f"tiles={tiles:4d} T={T:6d} K={4*T*D/1e6:7.1f} MB  roundtrip {ms*1e3:8.1f} us  "
          f"per K-block per CTA {ms*1e3/kb:6.3f} us  {gbs:7.1f} GB/s", flush=True)
    del K, Kq, Kh, ws
