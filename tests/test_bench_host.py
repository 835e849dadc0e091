"""Host logic of bench.py (no GPU): the per-step libkvq launch count it reports as gpu_launches follows the
path the step takes (csrc/: scales, prep, tensor-core pass, split_combine, reduction, exchange kernels)."""
import importlib.util
import os
import types

import pytest

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.fixture()
def b200(monkeypatch):
    monkeypatch.setattr(torch.cuda, "current_device", lambda: 0)
    monkeypatch.setattr(torch.cuda, "get_device_properties", lambda d: types.SimpleNamespace(multi_processor_count=148))


def args(fmt="int8", pipeline="fused"):
    return types.SimpleNamespace(format=fmt, pipeline=pipeline)


PEER = "peer (CUDA-IPC peer memory, libkvq kvq_comm_from_peer; no NCCL)"
NCCL = "nccl (libkvq kvq_comm_t)"


@pytest.mark.parametrize("rows,comm,kind,expect", [
    (131072, None, None, 5),        # one GPU: colmax, finalize, prep, attn_tc<2>, reduce (writes the result)
    (131072, object(), PEER, 6),    # fused colmax+exchange+finalize; + metric exchange + metrics_finalize
    (131072, object(), NCCL, 6),    # colmax, finalize, prep, attn, reduce, metrics_finalize (NCCL not counted)
    (65536, object(), PEER, 7),     # 2-rank shard: 512 tiles = 3 waves + 46% -> balanced tail, + split_combine
    (32768, object(), PEER, 6),     # 4-rank shard: 1.73 waves -> whole tiles
    (16384, object(), PEER, 6),     # 8-rank shard: one wave -> whole tiles
])
def test_fused_step_launch_count(bench, b200, rows, comm, kind, expect):
    assert bench.launches_per_step(args(), comm, kind, rows, 8192) == expect


def test_separate_and_format_launch_counts(bench, b200):
    # scales (2) + quantize + dequantize + metrics (qsplit, attn_tc<0>, reduce)
    assert bench.launches_per_step(args(pipeline="separate"), None, None, 131072, 8192) == 7
    # scales (2) + the format's fused quantize+dequantize + metrics (3)
    assert bench.launches_per_step(args(fmt="e4m3"), None, None, 131072, 8192) == 6
