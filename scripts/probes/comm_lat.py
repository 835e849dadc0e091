"""Latency of the step's collectives at world 1 (torchrun --nproc-per-node 1): the metric exchange
(kvq_error_metrics_async at a tiny shape) and the scale exchange, peer-backed vs NCCL communicator."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2601_04719_b200 import kvq  # noqa: E402
from paper_2601_04719_b200.dist import make_comm, make_peer  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
T, D, nq = 1024, 128, 64
K = kvq.kvq_synth_fill(T, D, seed=42)
Q = kvq.kvq_synth_fill(nq, D, seed=43)
s = kvq.kvq_compute_scales(K)
Kh = kvq.kvq_dequantize(kvq.kvq_quantize(K, s), s)
ws = torch.empty(kvq.kvq_error_metrics_workspace_size(T, D, nq), dtype=torch.uint8, device="cuda")
mout = torch.empty(kvq.METRICS_BYTES, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
peer = make_peer(0, 1, D)
comms = {"none": None, "nccl": make_comm(0, 1), "peer": kvq.Comm.from_peer(peer)}


def t(fn, n=200):
    for _ in range(20):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(n):
        fn()
    b.record(st)
    b.synchronize()
    return round(a.elapsed_time(b) / n * 1000, 2)


for name, c in comms.items():
    m = t(lambda: kvq.kvq_error_metrics_async(K, Kh, Q, s, out_dev=mout, workspace=ws, comm=c, stream=st))
    sc = t(lambda: kvq.kvq_compute_scales(K, s, comm=c, stream=st))
    print(f"{name}: error_metrics_async {m} us/call, compute_scales {sc} us/call", flush=True)
torch.cuda.synchronize()
comms["peer"].destroy()
comms["nccl"].destroy()
peer.destroy()
dist.destroy_process_group()
