#!/usr/bin/env python
"""Write tests/golden/oracle_attn.json: the oracle's attention-score error (P:24,
P:479-481; readings Q10/Q11: raw dot products, nq = 64 seeded queries, mean over
ALL T rows) for the BASELINE configs C1-C4, which the SURVEY appendix leaves
blank for C3/C4.  Calls only oracle/ (plain C, fp64): Alg. 1 over the whole
matrix, then quantize / dequantize / attention sums per row block.  The row
blocks run in parallel processes; their fp64 partial sums are added in block
order (the oracle's sequential sum differs only by rounding, ~1e-15 relative).

    python scripts/oracle_goldens.py [--procs 8]
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

CONFIGS = {"C1": (1024, 128), "C2": (8192, 1024), "C3": (32768, 8192), "C4": (131072, 8192)}
NQ = 64
BLOCK = 2048


def _absmax(args):
    T, D, r0 = args
    m = np.zeros(D, dtype=np.float32)
    oracle.absmax_rows(oracle.fill(min(BLOCK, T - r0), D, oracle.SEED_K, oracle.DIST_UNIFORM, r0), m)
    return m


def _attn(args):
    T, D, r0, s = args
    K = oracle.fill(min(BLOCK, T - r0), D, oracle.SEED_K, oracle.DIST_UNIFORM, r0)
    Kh = oracle.dequantize(oracle.quantize(K, s), s)
    Q = oracle.fill(NQ, D, oracle.SEED_Q)
    return oracle.attention_abs_sum(Q, K, Kh)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "oracle_attn.json"))
    args = ap.parse_args()
    oracle.build()
    res = {"_source": ("scripts/oracle_goldens.py: oracle/ only (plain C, fp64), seed_K=42, seed_Q=43, nq=64, "
                       "mean of |S - S'| over all (query, row) pairs (P:24, P:479-481; readings Q10, Q11)")}
    with mp.get_context("fork").Pool(args.procs) as pool:
        for name, (T, D) in CONFIGS.items():
            t0 = time.time()
            starts = list(range(0, T, BLOCK))
            m = np.zeros(D, dtype=np.float32)
            for part in pool.map(_absmax, [(T, D, r0) for r0 in starts]):
                m = np.maximum(m, part)  # Eq. 6: the max is order-free
            s = oracle.scales_from_absmax(m)
            sums = pool.map(_attn, [(T, D, r0, s) for r0 in starts])
            total = 0.0
            for x in sums:
                total += x
            res[name] = {"T": T, "D": D, "nq": NQ, "attn_abs_sum": total, "attn_mean_abs": total / (NQ * T)}
            print(name, res[name], f"{time.time() - t0:.1f} s", flush=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
