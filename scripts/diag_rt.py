"""Diagnose kvq_roundtrip vs the separate kernels at growing T."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_04719_b200 import kvq
D = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
for T in (1000, 1024, 2048, 4096, 8192, 16384):
    Kd = kvq.kvq_synth_fill(T, D, seed=42)
    Qd = kvq.kvq_synth_fill(64, D, seed=43)
    s = kvq.kvq_compute_scales(Kd)
    q1 = kvq.kvq_quantize(Kd, s)
    k1 = kvq.kvq_dequantize(q1, s)
    for rep in range(2):
        q2, k2, out = kvq.kvq_roundtrip(Kd, s, Qd)
        torch.cuda.synchronize()
        dq = (q1 != q2)
        dk = (k1.view(torch.int32) != k2.view(torch.int32))
        nq_bad, nk_bad = int(dq.sum()), int(dk.sum())
        msg = f"T={T} rep={rep} code mismatches={nq_bad} khat mismatches={nk_bad}"
        if nq_bad or nk_bad:
            idx = torch.nonzero(dq | dk)
            rows = torch.unique(idx[:, 0])
            cols = torch.unique(idx[:, 1])
            msg += f" rows[{rows.numel()}]={rows[:8].tolist()} cols[{cols.numel()}]={cols[:8].tolist()}"
            r, c = idx[0].tolist()
            msg += f" first=({r},{c}) q1={int(q1[r,c])} q2={int(q2[r,c])} k1={float(k1[r,c])} k2={float(k2[r,c])} K={float(Kd[r,c])}"
        print(msg, flush=True)
