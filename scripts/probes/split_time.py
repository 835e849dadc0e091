"""Roundtrip (kvq_compute_scales + kvq_roundtrip) device time vs the K-block split (KVQ_TC_SPLIT) for token
shards of C4 (T = 131072 / N rows, D = 8192) and C2/C3."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2601_04719_b200 import kvq  # noqa: E402

st = torch.cuda.current_stream()
for T, D in [(16384, 8192), (32768, 8192), (65536, 8192), (8192, 1024), (131072, 8192)]:
    K = kvq.kvq_synth_fill(T, D, seed=42)
    Q = kvq.kvq_synth_fill(64, D, seed=43)
    s = kvq.kvq_compute_scales(K)
    Kq = torch.empty(T, D, dtype=torch.int8, device="cuda")
    Kh = torch.empty(T, D, dtype=torch.float32, device="cuda")
    mout = torch.empty(kvq.METRICS_BYTES, dtype=torch.uint8, device="cuda")
    res = {}
    for sp in ["auto", "1", "2", "4", "8"]:
        if sp == "auto":
            os.environ.pop("KVQ_TC_SPLIT", None)
        else:
            os.environ["KVQ_TC_SPLIT"] = sp
        ws = torch.empty(kvq.kvq_roundtrip_workspace_size(T, D, 64), dtype=torch.uint8, device="cuda")
        ts = []
        for i in range(25):
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record(st)
            kvq.kvq_compute_scales(K, s, stream=st)
            b.record(st)
            kvq.kvq_roundtrip(K, s, Q, Kq, Kh, out_dev=mout, workspace=ws, stream=st)
            c.record(st)
            c.synchronize()
            if i >= 5:
                ts.append(b.elapsed_time(c))
        res[sp] = round(statistics.median(ts), 4)
    os.environ.pop("KVQ_TC_SPLIT", None)
    print(T, D, "roundtrip ms by split:", res, flush=True)
    del K, Kq, Kh
    torch.cuda.empty_cache()
