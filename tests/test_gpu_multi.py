"""GPU, one process per device (PAPER.md:566 multi-GPU future work): the token-sharded step
across 2 / 4 / 8 GPUs with both communicators (the library's NCCL one and the CUDA-IPC peer-memory one),
checked against the CPU oracle.  Collected everywhere; skipped unless at least `world` GPUs are visible
(the round-end box has one, an 8-GPU node runs all of them).

* C2 (8192 x 1024, nq = 64): every rank's scales equal the oracle's (global column max, a7), the shards
  concatenated in rank order equal the oracle's codes and K_hat bit for bit, and the metrics (all-reduced
  over the ranks) agree with the oracle's L2 / max-abs / attention error.
* C4 (131072 x 8192) at the largest world: scales equal the SURVEY appendix golden, every rank's codes and
  K_hat equal the oracle's on its own rows (chunked), L2 / max-abs agree with the goldens.
* "nvls": the peer exchange with the a7 max read through NVLS multicast (multimem.ld_reduce in the NVSwitch)
  when every rank can map it, else every rank keeps P2P (the same results either way).
* bench.py --gpus N (self-launch under torch.distributed.run) prints one line with n_gpus = N for both
  communicators, and the two give the same fidelity metrics.
"""
import hashlib
import json
import os
import socket
import subprocess
import sys
import traceback

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0

C2 = (8192, 1024, 64)
C4 = (131072, 8192, 64)
C4_SCALES_SHA16 = "97ddf41b62a0d957"  # SURVEY.md appendix (numpy, independent of both paths)
C4_L2 = 74.48112853965452
C4_MAX_ABS = 0.0039370059967041016


SHARE = os.environ.get("KVQ_TEST_SHARE_GPU") == "1"  # harness check on one GPU: ranks time-slice cuda:0


def _need(world, comm_kind="nccl"):
    if NGPU >= world or (SHARE and NGPU >= 1 and comm_kind in ("peer", "nvls")):
        return
    pytest.skip(f"needs {world} GPUs, {NGPU} visible")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, out_dir, comm_kind, cfg, check_rows):
    sys.path.insert(0, ROOT)
    res_path = os.path.join(out_dir, f"rank{rank}.npz")
    try:
        import torch.distributed as dist

        from paper_2601_04719_b200 import kvq
        from paper_2601_04719_b200.dist import enable_nvls, make_comm, make_peer, shard_rows
        dev = torch.device("cuda", rank % torch.cuda.device_count())
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        T, D, nq = cfg
        row0, rows = shard_rows(T, world, rank)
        K = kvq.kvq_synth_fill(rows, D, row0=row0, seed=42, device=dev)
        Q = kvq.kvq_synth_fill(nq, D, seed=43, device=dev)
        peer = None
        nvls = False
        if comm_kind in ("peer", "nvls"):
            peer = make_peer(rank, world, D)
            if comm_kind == "nvls":
                nvls = enable_nvls(peer, rank, world)  # False: no multicast here, the P2P exchange is kept
            comm = kvq.Comm.from_peer(peer)
        else:
            comm = make_comm(rank, world)
        s = kvq.kvq_compute_scales(K, comm=comm)
        q, kh, out = kvq.kvq_roundtrip(K, s, Q, comm=comm)
        m = kvq.metrics_from_device(out)
        # the separate calls (a3, a4, then a5 + a6 with the metric exchange)
        q2 = kvq.kvq_quantize(K, s)
        kh2 = kvq.kvq_dequantize(q2, s)
        m2 = kvq.kvq_error_metrics(K, kh2, Q, s, comm=comm)
        torch.cuda.synchronize()
        same = bool(torch.equal(q, q2) and torch.equal(kh.view(torch.int32), kh2.view(torch.int32)))
        res = dict(scales=s.cpu().numpy(), same=np.array(same), row0=np.array(row0), rows=np.array(rows),
                   nvls=np.array(nvls),
                   metrics=np.array([m["l2"], m["max_abs"], m["attn_mean_abs"]]),
                   metrics2=np.array([m2["l2"], m2["max_abs"], m2["attn_mean_abs"]]))
        if check_rows:
            # the oracle on this rank's own rows (chunked), with the global scales just computed
            import oracle as orc
            sc = res["scales"]
            bad = 0
            for c0 in range(0, rows, check_rows):
                n = min(check_rows, rows - c0)
                Ko = orc.fill(n, D, orc.SEED_K, row0=row0 + c0)
                qo = orc.quantize(Ko, sc)
                ko = orc.dequantize(qo, sc)
                bad += int(not np.array_equal(q[c0:c0 + n].cpu().numpy(), qo))
                bad += int(not np.array_equal(kh[c0:c0 + n].cpu().numpy().view(np.uint32), ko.view(np.uint32)))
            res["bad_chunks"] = np.array(bad)
        else:
            res["q"] = q.cpu().numpy()
            res["kh"] = kh.cpu().numpy()
        torch.cuda.synchronize()
        dist.barrier()
        comm.destroy()
        if peer is not None:
            peer.destroy()
        dist.destroy_process_group()
        np.savez(res_path, **res)
    except Exception:  # noqa: BLE001
        with open(os.path.join(out_dir, f"rank{rank}.err"), "w") as f:
            f.write(traceback.format_exc())
        raise


def _run(world, comm_kind, cfg, tmp_path, check_rows=0, timeout=900):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, str(tmp_path), comm_kind, cfg, check_rows))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout)
    for p in procs:
        if p.is_alive():
            p.kill()
    errs = [open(tmp_path / f).read() for f in os.listdir(tmp_path) if f.endswith(".err")]
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("comm_kind", ["nccl", "peer", "nvls"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_c2_matches_oracle(orc, tmp_path, world, comm_kind):
    _need(world, comm_kind)
    T, D, nq = C2
    res = _run(world, comm_kind, C2, tmp_path)
    Ko = orc.fill(T, D)
    so, qo, kho = orc.roundtrip(Ko)
    assert len({bool(r["nvls"]) for r in res}) == 1, "NVLS must be on for all ranks or for none"
    for r in res:
        assert np.array_equal(r["scales"].view(np.uint32), so.view(np.uint32)), "a7: global scales on every rank"
        assert bool(r["same"]), "kvq_roundtrip and the separate calls disagree"
    assert sum(int(r["rows"]) for r in res) == T
    q = np.concatenate([r["q"] for r in res])
    kh = np.concatenate([r["kh"] for r in res])
    assert np.array_equal(q, qo)
    assert np.array_equal(kh.view(np.uint32), kho.view(np.uint32))
    l2 = orc.l2_error(Ko, kho)
    mx = orc.max_abs_error(Ko, kho)
    attn = orc.attention_error(orc.fill(nq, D, 43), Ko, kho)
    for r in res:  # every rank holds the same (all-reduced) metrics, from both paths
        for key in ("metrics", "metrics2"):
            l2g, mxg, attng = r[key]
            assert abs(l2g - l2) <= 1e-5 * l2
            assert mxg == mx
            assert abs(attng - attn) <= 1e-5 * attn


@pytest.mark.timeout(2400)
@pytest.mark.parametrize("comm_kind", ["nccl", "peer", "nvls"])
def test_sharded_c4_matches_goldens_and_oracle(tmp_path, comm_kind):
    world = max(w for w in (2, 4, 8) if w <= max(NGPU, 2))
    _need(world, comm_kind)
    res = _run(world, comm_kind, C4, tmp_path, check_rows=8192, timeout=2000)
    for r in res:
        assert hashlib.sha256(r["scales"].tobytes()).hexdigest()[:16] == C4_SCALES_SHA16
        assert bool(r["same"])
        assert int(r["bad_chunks"]) == 0
        l2g, mxg, _ = r["metrics"]
        assert abs(l2g - C4_L2) <= 1e-5 * C4_L2
        assert mxg == C4_MAX_ABS


@pytest.mark.timeout(900)
@pytest.mark.parametrize("world", [2, 8])
def test_bench_gpus_n_self_launch(world):
    """`python bench.py --gpus N` (no torchrun) runs N ranks and reports n_gpus = N; peer and NCCL
    exchanges give the same fidelity metrics."""
    _need(world)
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    fid = {}
    for comm in ("peer", "nccl"):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(world), "--config", "C2",
                            "--steps", "5", "--warmup", "3", "--no-e2e", "--no-cpu", "--comm", comm],
                           capture_output=True, text=True, env=env, timeout=800, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-3000:]
        lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
        assert len(lines) == 1, r.stdout
        line = lines[0]
        assert line["n_gpus"] == world and line["config"]["comm"].startswith(comm)
        fid[comm] = line["fidelity"]
    assert fid["peer"]["max_abs"] == fid["nccl"]["max_abs"]
    assert abs(fid["peer"]["l2"] - fid["nccl"]["l2"]) <= 1e-12 * fid["nccl"]["l2"]
    assert abs(fid["peer"]["attn_mean_abs"] - fid["nccl"]["attn_mean_abs"]) <= 1e-9 * fid["nccl"]["attn_mean_abs"]
