import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle
from paper_2601_04719_b200 import kvq
for (T, D, nq) in [(128, 64, 64), (1000, 1024, 64), (300, 128, 17), (131, 160, 9)]:
    K = oracle.fill(T, D, 6, 1); so, qo, kho = oracle.roundtrip(K); Q = oracle.fill(nq, D, 43)
    Kd = torch.from_numpy(K).cuda(); s = kvq.kvq_compute_scales(Kd)
    Kq, Kh, out = kvq.kvq_roundtrip(Kd, s, torch.from_numpy(Q).cuda()); m = kvq.metrics_from_device(out)
    a = oracle.attention_error(Q, K, kho)
    print(T, D, nq, "codes", np.array_equal(Kq.cpu().numpy(), qo), "khat", np.array_equal(Kh.cpu().numpy().view(np.uint32), kho.view(np.uint32)),
          "attn", m["attn_mean_abs"], a, abs(m["attn_mean_abs"] - a) / a, "maxabs", m["max_abs"], flush=True)
