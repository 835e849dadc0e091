#!/usr/bin/env python
"""Write tests/golden/oracle_c5.json: SHA-256 of the oracle's scales, codes and K_hat (Alg. 1, Eq. 6/7/8;
readings Q1-Q8) at the extremes of BASELINE config C5 (the L2-resident vs streaming sweep, 2^20..2^30
elements at head_dim 128/1024/8192): 2^30 elements at D = 128 and D = 1024 (streaming, 4.3 GB of K) and
2^24 at D = 1024 and D = 8192 (the single-pass / two-pass crossover).  Calls only oracle/ (plain C): the
column maxima over row blocks (Eq. 6 is order-free), then quantize / dequantize per row block, the bytes
hashed in row order (the SHA of the whole row-major matrix).  Row blocks run in worker processes.

    python scripts/oracle_c5_goldens.py [--procs 8]
"""
import argparse
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

SHAPES = {"2^30 x D128": (1 << 23, 128), "2^30 x D1024": (1 << 20, 1024), "2^24 x D1024": (1 << 14, 1024),
          "2^24 x D8192": (1 << 11, 8192)}
BLOCK_ELEMS = 1 << 24  # 64 MB of fp32 per block


def _absmax(args):
    rows, D, r0 = args
    m = np.zeros(D, dtype=np.float32)
    oracle.absmax_rows(oracle.fill(rows, D, oracle.SEED_K, oracle.DIST_UNIFORM, r0), m)
    return m


def _qdq(args):
    rows, D, r0, s = args
    K = oracle.fill(rows, D, oracle.SEED_K, oracle.DIST_UNIFORM, r0)
    q = oracle.quantize(K, s)
    kh = oracle.dequantize(q, s)
    return q.tobytes(), kh.tobytes()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "oracle_c5.json"))
    args = ap.parse_args()
    oracle.build()
    res = {"_source": ("scripts/oracle_c5_goldens.py: oracle/ only (plain C), seed_K = 42, uniform lattice "
                       "(SURVEY §8(d)); sha256 of the raw little-endian row-major bytes")}
    with mp.get_context("fork").Pool(args.procs) as pool:
        for name, (T, D) in SHAPES.items():
            t0 = time.time()
            br = max(1, BLOCK_ELEMS // D)
            blocks = [(min(br, T - r0), D, r0) for r0 in range(0, T, br)]
            m = np.zeros(D, dtype=np.float32)
            for part in pool.imap(_absmax, blocks):
                m = np.maximum(m, part)  # Eq. 6: the max is order-free
            s = oracle.scales_from_absmax(m)
            hq, hk = hashlib.sha256(), hashlib.sha256()
            for qb, kb in pool.imap(_qdq, [(rows, D, r0, s) for rows, D, r0 in blocks]):  # in row order
                hq.update(qb)
                hk.update(kb)
            res[name] = {"T": T, "D": D, "scales_sha256": hashlib.sha256(s.tobytes()).hexdigest(),
                         "codes_sha256": hq.hexdigest(), "k_hat_sha256": hk.hexdigest()}
            print(name, res[name], f"{time.time() - t0:.1f} s", flush=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
