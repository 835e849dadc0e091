"""Roundtrip ring depth (KVQ_RT_STAGES) A/B: in-step timing and bit-identical outputs vs the default depth."""
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


def run(n=40):
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n)]
    for i in range(n + 5):
        e = ev[i - 5] if i >= 5 else None
        if e: e[0].record(st)
        kvq.kvq_compute_scales(K, s, stream=st)
        if e: e[1].record(st)
        kvq.kvq_roundtrip(K, s, Q, Kq, Kh, out_dev=mout, workspace=ws, stream=st)
        if e: e[2].record(st)
    torch.cuda.synchronize()
    c = statistics.median(a.elapsed_time(b) for a, b, _ in ev)
    r = statistics.median(b.elapsed_time(x) for _, b, x in ev)
    return round(c, 4), round(r, 4)


os.environ["KVQ_RT_STAGES"] = "8"
run(3)
ref = (Kq.clone(), Kh.clone(), mout.clone())
for rep in range(2):
    for stg in sys.argv[1:] or ["4", "5", "6", "8"]:
        os.environ["KVQ_RT_STAGES"] = stg
        t = run()
        same = all(torch.equal(a, b) for a, b in zip(ref, (Kq, Kh, mout)))
        print(f"stages={stg} step (colmax, roundtrip) ms: {t}  outputs identical to 8 stages: {same}", flush=True)
