#!/usr/bin/env python
"""NEXT-1 / NEXT-3 fidelity comparison: INT8 (the paper's method) vs FP8 E4M3, INT4 and INT2 per-channel
quantization of the same key matrices, through the same fidelity checks (a5, a6:
L2, max-abs, mean |Q.K^T - Q.K_hat^T| with nq = 64).  Both paths are parity-tested
bit-exact against the oracle (tests/test_gpu_parity.py, tests/test_gpu_fp8.py);
this script only runs the GPU path on the BASELINE configs and prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_04719_b200 import kvq  # noqa: E402

CONFIGS = {"C1": (1024, 128), "C2": (8192, 1024), "C3": (32768, 8192), "C4": (131072, 8192)}
out = {}
for name, (T, D) in CONFIGS.items():
    row = {}
    for dist, dname in ((kvq.DIST_UNIFORM, "uniform"), (kvq.DIST_OUTLIER, "outlier_channels")):
        K = kvq.kvq_synth_fill(T, D, seed=42, dist=dist)
        Q = kvq.kvq_synth_fill(64, D, seed=43)
        res = {}
        s8 = kvq.kvq_compute_scales(K)
        q8, kh8 = kvq.kvq_quantize_dequantize(K, s8)
        res["int8"] = kvq.kvq_error_metrics(K, kh8, Q, s8)
        del q8, kh8
        sf = kvq.kvq_compute_scales_fmt(K, kvq.FMT_E4M3)
        qf, khf = kvq.kvq_quantize_e4m3(K, sf, want_khat=True)
        res["e4m3"] = kvq.kvq_error_metrics(K, khf, Q, sf)
        del qf, khf
        for bits, fmt in ((4, kvq.FMT_INT4), (2, kvq.FMT_INT2)):
            sb = kvq.kvq_compute_scales_fmt(K, fmt)
            pb, khb = kvq.kvq_quantize_packed(K, sb, bits, want_khat=True)
            res[f"int{bits}"] = kvq.kvq_error_metrics(K, khb, Q, sb)
            del pb, khb
        del K
        torch.cuda.empty_cache()
        row[dname] = {fmt: {k: m[k] for k in ("l2", "max_abs", "attn_mean_abs")} for fmt, m in res.items()}
    out[name] = {"T": T, "D": D, **row}
print(json.dumps(out))
