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
    monkeypatch.setattr(torch.cuda, "get_device_properties",
                        lambda d: types.SimpleNamespace(multi_processor_count=148, L2_cache_size=126 << 20))


def args(fmt="int8", pipeline="fused"):
    return types.SimpleNamespace(format=fmt, pipeline=pipeline)


PEER = "peer (CUDA-IPC peer memory, libkvq kvq_comm_from_peer; no NCCL)"
NCCL = "nccl (libkvq kvq_comm_t)"


@pytest.mark.parametrize("rows,comm,kind,expect", [
    (131072, None, None, 4),        # one GPU: colmax, finalize, prep, attn_tc<2> (its last CTA reduces the partials)
    (131072, object(), PEER, 5),    # fused colmax+exchange+finalize; prep, attn; + metric exchange + metrics_finalize
    (131072, object(), NCCL, 5),    # colmax, finalize, prep, attn, metrics_finalize (NCCL not counted)
    (65536, object(), PEER, 7),     # 2-rank shard: 512 tiles = 3 waves + 46% -> balanced tail, + split_combine + reduce
    (32768, object(), PEER, 7),     # 4-rank shard: 1.73 waves -> 1 whole wave + 108 tiles in 4 pieces, + combine + reduce
    (16384, object(), PEER, 5),     # 8-rank shard: one wave -> whole tiles
])
def test_fused_step_launch_count(bench, b200, rows, comm, kind, expect):
    assert bench.launches_per_step(args(), comm, kind, rows, 8192) == expect


@pytest.mark.parametrize("rows,comm,kind,expect", [
    (131072, None, None, 5),        # one GPU: colmax, finalize, prep, rt64_kernel, reduce (writes the result)
    (65536, object(), PEER, 6),     # 2-rank shard: 1024 64-row tiles = 6.9 waves -> whole tiles
    (32768, object(), PEER, 7),     # 4-rank shard: 512 tiles = 3 waves + 68 tiles in 2 pieces, + split_combine64
    (16384, object(), PEER, 7),     # 8-rank shard: 256 tiles = 1 wave + 108 tiles in 4 pieces, + split_combine64
])
def test_fused_step_launch_count_rt64(bench, b200, monkeypatch, rows, comm, kind, expect):
    """The opt-in 64-row roundtrip kernel (KVQ_TC_RT64=1, rt64_kernel)."""
    monkeypatch.setenv("KVQ_TC_RT64", "1")
    assert bench.launches_per_step(args(), comm, kind, rows, 8192) == expect


def test_separate_and_format_launch_counts(bench, b200):
    # scales (2) + quantize + dequantize + metrics (qsplit, attn_tc<0>, reduce)
    assert bench.launches_per_step(args(pipeline="separate"), None, None, 131072, 8192) == 7
    # scales (2) + the format's fused quantize+dequantize + metrics (3)
    assert bench.launches_per_step(args(fmt="e4m3"), None, None, 131072, 8192) == 6


def test_gpus_n_self_launches_under_torchrun(bench):
    """`bench.py --gpus 2` without torchrun re-launches itself with 2 processes (never a silent 1-GPU run)."""
    seen = []
    rc = bench.self_launch(2, ["--gpus", "2", "--steps", "3"], device_count=8, run=lambda c: seen.append(c) or 0)
    assert rc == 0 and len(seen) == 1
    cmd = seen[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=2" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "2", "--steps", "3"][-3:] and cmd[-4] == "--gpus"


def test_gpus_n_fails_loudly_without_enough_gpus(bench, capsys):
    rc = bench.self_launch(4, ["--gpus", "4"], device_count=1, run=lambda c: pytest.fail("must not launch"))
    assert rc != 0
    assert "needs 4 visible GPUs, found 1" in capsys.readouterr().err


def test_gpus_n_cli_exits_nonzero_on_cpu_box():
    """End to end through the CLI on this GPU-less box: exit code != 0 and no JSON line claiming n_gpus 1."""
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0
    assert '"n_gpus"' not in r.stdout


def test_cpu_report_per_pass(bench):
    t = {"scales": 1.0, "quantize": 2.0, "dequantize": 1.0, "recon_errors": 1.0, "attention": 5.0}
    r = bench.cpu_report(t, 400, steps=2)
    assert r["value"] == 400 * 2 / 4.0
    assert r["full_step_elements_per_s"] == 400 * 2 / 10.0
    assert r["per_pass_s"]["attention"] == 2.5


def test_plan_tail_cases(bench):
    """The tail plan (attn_tc.cu tc_plan_tail) at the C4 shard sizes on 148 SMs (D = 8192: 64 units per tile)."""
    assert not bench.plan_tail(1024, 64, 148)["split"]                       # 1 rank: 6.92 waves, whole
    assert bench.plan_tail(512, 64, 148) == {"split": True, "grid": 148, "whole": 3, "rt": 68, "pieces": 2}
    assert bench.plan_tail(256, 64, 148) == {"split": True, "grid": 148, "whole": 1, "rt": 108, "pieces": 4}
    assert not bench.plan_tail(128, 64, 148)["split"]                        # 8 ranks: under one wave
    assert bench.plan_tail(64, 8, 148) == {"split": True, "grid": 148, "whole": 0, "rt": 64, "pieces": 2}  # C2
    assert not bench.plan_tail(8, 1, 148)["split"]                           # C1: one unit per tile


def test_step_pipeline_launch_counts(bench, b200):
    a = types.SimpleNamespace(format="int8", pipeline="step")
    assert bench.launches_per_step(a, None, None, 1024, 128) == 1        # C1: one cooperative launch
    assert bench.launches_per_step(a, None, None, 8192, 1024) == 3       # C2: fused pass (Q split inside) + combine + reduce
    assert bench.launches_per_step(a, None, None, 131072, 8192) == 4     # C4: the two calls


def test_all_cores_oracle_line(bench):
    """SURVEY §8(d)'s optional all-cores CPU line: the unchanged oracle functions on row blocks in threads; the
    combined column maxima give bit-identical scales to the one-core oracle."""
    import numpy as np

    import oracle
    cfg = {"D": 256, "nq": 8, "T": 1000, "name": "t"}
    t, n = bench.oracle_step_all_cores(cfg, 300, 4)
    assert n == 300 * 256 and set(t) == {"scales", "quantize", "dequantize"} and all(v >= 0 for v in t.values())
    for dist in (0, 1):  # uniform and outlier-channel keys
        K = oracle.fill(300, 256, oracle.SEED_K, dist)
        blocks = [np.ascontiguousarray(b) for b in np.array_split(K, 4)]
        s = np.maximum.reduce([oracle.compute_scales(b) for b in blocks])  # fl32(m/127) is monotonic in m
        assert np.array_equal(s.view(np.uint32), oracle.compute_scales(K).view(np.uint32))
