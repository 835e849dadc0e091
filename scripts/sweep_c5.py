#!/usr/bin/env python
"""BASELINE.json configs[4] (C5): L2-resident vs streaming sweep, 1M-1B elements at
head_dim 128 / 1024 / 8192, single-pass fused (kvq_quantize_fused: one cooperative
launch) vs two-pass (kvq_compute_scales + kvq_quantize_dequantize), each with the
L2 cold (a 512 MB buffer written between iterations, outside the timed events)
and warm.  Bytes per element are the algorithmic ones: 4 (a1) + 4 + 5 (a3+a4 fused)
= 13 for the two-pass pipeline; the single pass moves 9 from HBM when K stays in L2.

    python scripts/sweep_c5.py [--out profiles/r01/sweep_c5] [--iters 10]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2601_04719_b200 import kvq  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "sweep_c5"))
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--kmin", type=int, default=20)
    ap.add_argument("--kmax", type=int, default=30)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    rows = []
    for D in (128, 1024, 8192):
        for k in range(a.kmin, a.kmax + 1):
            N = 1 << k
            T = N // D
            if T < 1:
                continue
            K = kvq.kvq_synth_fill(T, D, seed=42, device=dev)
            s = torch.empty(D, dtype=torch.float32, device=dev)
            q = torch.empty((T, D), dtype=torch.int8, device=dev)
            kh = torch.empty((T, D), dtype=torch.float32, device=dev)
            ws = torch.empty(kvq.load().kvq_quantize_fused_workspace_size(T, D), dtype=torch.uint8, device=dev)

            def two_pass():
                kvq.kvq_compute_scales(K, s, stream=stream)
                kvq.kvq_quantize_dequantize(K, s, q, kh, stream=stream)

            single_flag = {}

            def single_pass():  # the cooperative kernel on every shape it supports
                os.environ["KVQ_FUSED_FORCE_SINGLE"] = "1"
                single_flag["v"] = kvq.kvq_quantize_fused(K, s, q, kh, workspace=ws, stream=stream)[3]
                del os.environ["KVQ_FUSED_FORCE_SINGLE"]

            def fused_auto():  # kvq_quantize_fused's own choice (single pass only while K is L2-resident)
                single_flag["auto"] = kvq.kvq_quantize_fused(K, s, q, kh, workspace=ws, stream=stream)[3]

            for name, fn in (("two_pass", two_pass), ("single_pass", single_pass), ("fused_auto", fused_auto)):
                for cold in (True, False):
                    for _ in range(3):
                        fn()
                    ts = []
                    for _ in range(a.iters):
                        if cold:
                            flush.fill_(1)
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        fn()
                        e1.record(stream)
                        e1.synchronize()
                        ts.append(e0.elapsed_time(e1))
                    ms = statistics.median(ts)
                    algo = 13 * N if name == "two_pass" else 13 * N  # same method bytes; see docstring
                    r = {"D": D, "T": T, "N": N, "pipeline": name, "l2": "cold" if cold else "warm",
                         "ms": ms, "elements_per_s": N / (ms * 1e-3), "algo_GBps_13B": algo / (ms * 1e-3) / 1e9,
                         "frac_of_measured_hbm": algo / (ms * 1e-3) / 1e9 / peak,
                         "single_pass_ran": (single_flag.get("v") if name == "single_pass" else
                                             single_flag.get("auto") if name == "fused_auto" else None),
                         "K_MB": 4 * N / 1e6}
                    rows.append(r)
                    print(json.dumps(r), flush=True)
            del K, q, kh, ws
            torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out + ".json", "w") as f:
        json.dump(rows, f, indent=1)
    with open(a.out + ".md", "w") as f:
        f.write("# C5 sweep: single-pass fused vs two-pass (a1..a4), B200, median of %d\n\n" % a.iters)
        f.write("GB/s use the method's 13 algorithmic bytes/element (4 for a1 + 9 for a3+a4) for both "
                "pipelines; above the HBM peak means L2 reuse.\n\n")
        f.write("`kvq_quantize_fused` (auto) runs the single pass only where K is L2-resident (D >= 256 and K <= 3/4 of "
                "the L2), else the two passes.\n\n")
        f.write("| D | N | K MB | L2 | two-pass ms | single-pass ms | two-pass GB/s | single-pass GB/s | speed-up | "
                "fused auto ms (path) |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|\n")
        for D in (128, 1024, 8192):
            for k in range(a.kmin, a.kmax + 1):
                for l2 in ("cold", "warm"):
                    sel = {r["pipeline"]: r for r in rows if r["D"] == D and r["N"] == 1 << k and r["l2"] == l2}
                    if len(sel) < 3:
                        continue
                    t2, t1, ta = sel["two_pass"], sel["single_pass"], sel["fused_auto"]
                    path = "single" if ta["single_pass_ran"] else "two-pass"
                    f.write(f"| {D} | 2^{k} | {t2['K_MB']:.0f} | {l2} | {t2['ms']:.4f} | {t1['ms']:.4f} | "
                            f"{t2['algo_GBps_13B']:.0f} | {t1['algo_GBps_13B']:.0f} | {t2['ms'] / t1['ms']:.2f} | "
                            f"{ta['ms']:.4f} ({path}) |\n")


if __name__ == "__main__":
    main()
