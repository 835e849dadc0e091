"""Per-rank step time of the C4 headline step on the shard a rank owns at N = 1, 2, 4, 8 (strong scaling:
T/N rows each), timed on one GPU.  Predicts the compute part of the multi-GPU efficiency:
eff(N) = t(1) / (N * t(T/N)); the exchange (a7 + metric partials) is not included.

    python scripts/probes/shard_time.py [--steps 100]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2601_04719_b200 import kvq  # noqa: E402
from paper_2601_04719_b200.dist import shard_rows  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--ns", default="1,2,4,8")
args = ap.parse_args()
T, D, nq = 131072, 8192, 64
st = torch.cuda.current_stream()
Q = kvq.kvq_synth_fill(nq, D, seed=43)
base = None
for N in [int(x) for x in args.ns.split(",")]:
    row0, rows = shard_rows(T, N, N - 1)  # the last rank's shard
    K = kvq.kvq_synth_fill(rows, D, row0=row0, seed=42)
    s = torch.empty(D, dtype=torch.float32, device="cuda")
    Kq = torch.empty((rows, D), dtype=torch.int8, device="cuda")
    Kh = torch.empty((rows, D), dtype=torch.float32, device="cuda")
    ws = torch.empty(kvq.kvq_roundtrip_workspace_size(rows, D, nq), dtype=torch.uint8, device="cuda")
    mout = torch.empty(kvq.METRICS_BYTES, dtype=torch.uint8, device="cuda")

    def step(ev=None):
        if ev:
            ev[0].record(st)
        kvq.kvq_compute_scales(K, s, stream=st)
        if ev:
            ev[1].record(st)
        kvq.kvq_roundtrip(K, s, Q, Kq, Kh, out_dev=mout, workspace=ws, stream=st)
        if ev:
            ev[2].record(st)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for i in range(args.steps):
        step(evs[i])
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    sc = statistics.median(e[0].elapsed_time(e[1]) for e in evs)
    rt = statistics.median(e[1].elapsed_time(e[2]) for e in evs)
    if base is None:
        base = ms
    print(f"N={N} rows={rows} tiles={(rows + 127) // 128} step {ms:.4f} ms (scales {sc:.4f}, roundtrip {rt:.4f}) "
          f"GB/s {13 * rows * D / ms / 1e6:.0f} predicted eff {base / (N * ms):.3f}", flush=True)
    del K, Kq, Kh, ws
    torch.cuda.empty_cache()
