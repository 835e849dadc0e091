#!/usr/bin/env python
"""NEXT-2 measurement: raw attention scores S = Q . K_hat^T (nq = 64) over the
C4 cache (131072 x 8192), either straight from the int8 codes
(kvq_scores_from_codes: int8 tensor cores, reads 1 B/key element) or from the fp32 reconstruction
(kvq_attention_scores on K_hat: 4 B/element).  Median of 20 event-timed runs."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_04719_b200 import kvq  # noqa: E402


def timeit(fn, iters=20):
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


T, D, nq = 131072, 8192, 64
K = kvq.kvq_synth_fill(T, D)
Q = kvq.kvq_synth_fill(nq, D, seed=43)
s = kvq.kvq_compute_scales(K)
q = kvq.kvq_quantize(K, s)
kh = kvq.kvq_dequantize(q, s)
del K
S = torch.empty((nq, T), dtype=torch.float32, device="cuda")
ws1 = torch.empty(kvq.load().kvq_scores_from_codes_workspace_size(D, nq), dtype=torch.uint8, device="cuda")
ws2 = torch.empty(kvq.load().kvq_attention_scores_workspace_size(D, nq), dtype=torch.uint8, device="cuda")
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
flops = 2.0 * nq * T * D
ms_codes = timeit(lambda: kvq.kvq_scores_from_codes(Q, q, s, S=S, workspace=ws1))
ms_fp32 = timeit(lambda: kvq.kvq_attention_scores(Q, kh, S=S, workspace=ws2))
# executed int8 tensor work: 4 digit planes x 64 queries = N 256 per 128x32 step
iops = 2.0 * 4 * 64 * T * D
hbm = peaks.get("hbm_gbs")
out = {
    "workload": "S = Q.K_hat^T, nq=64, T=131072, D=8192 (C4)",
    "codes_i8_tc": {"ms": ms_codes, "hbm_GBps": T * D / (ms_codes * 1e-3) / 1e9,
                    "frac_of_hbm": (T * D / (ms_codes * 1e-3) / 1e9) / hbm if hbm else None,
                    "algo_TFLOPs": flops / (ms_codes * 1e-3) / 1e12,
                    "executed_int8_TOPs_4_digits": iops / (ms_codes * 1e-3) / 1e12,
                    "frac_of_int8_peak_executed": iops / (ms_codes * 1e-3) / 1e12 / (2 * peaks["bf16_tflops"])},
    "fp32_tf32x3_tc": {"ms": ms_fp32, "hbm_GBps": 4 * T * D / (ms_fp32 * 1e-3) / 1e9,
                       "algo_TFLOPs": flops / (ms_fp32 * 1e-3) / 1e12},
    "speedup_codes_vs_fp32": ms_fp32 / ms_codes,
}
print(json.dumps(out))
