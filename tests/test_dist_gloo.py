"""Multi-process (world size 2, gloo, CPU) tests of the token-sharding path
(DESIGN.md §7).  The GPU build does the exchange inside
libkvq.so over NCCL; here the same host plumbing (paper_2601_04719_b200.dist:
row partition, unique-id broadcast, max-over-ranks timing) runs over gloo, and
the sharding algebra is checked with the oracle standing in for the kernels:
local column max -> all-reduce MAX of the abs-bit patterns -> /127 gives the
unsharded scales bit-exactly, shard codes concatenate to the unsharded codes,
and summed / maxed metric partials reproduce the unsharded metrics."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_04719_b200.dist import broadcast_bytes, max_over_ranks, shard_rows, sum_over_ranks

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, T, D, nq, dist_kind, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        row0, rows = shard_rows(T, world, rank)
        K = oracle.fill(rows, D, oracle.SEED_K, dist_kind, row0)
        # a1 on the shard, then the a7 exchange: MAX over ranks of the uint32 abs bits
        m = np.zeros(D, dtype=np.float32)
        oracle.absmax_rows(K, m)
        bits = torch.from_numpy(m.view(np.int32).copy())  # abs bits <= 0x7fffffff: int32 order == float order
        dist.all_reduce(bits, op=dist.ReduceOp.MAX)
        s = oracle.scales_from_absmax(bits.numpy().view(np.float32).copy())
        q = oracle.quantize(K, s)
        Kh = oracle.dequantize(q, s)
        ss, mx = oracle.recon_errors(K, Kh)
        Q = oracle.fill(nq, D, oracle.SEED_Q)
        attn = oracle.attention_abs_sum(Q, K, Kh)
        # metric combination exactly as kvq_error_metrics with a communicator does it
        sums = torch.tensor([ss, attn, rows * D, nq * rows], dtype=torch.float64)
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        maxes = torch.tensor([mx], dtype=torch.float64)
        dist.all_reduce(maxes, op=dist.ReduceOp.MAX)
        # gather the shard codes on rank 0
        qt = torch.from_numpy(q.astype(np.int32).reshape(-1))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([qt.numel()]))
        mxn = int(max(x.item() for x in sizes))
        buf = torch.zeros(mxn, dtype=torch.int32)
        buf[:qt.numel()] = qt
        bufs = [torch.zeros(mxn, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(bufs, buf)
        # host helpers used by bench.py
        uid = broadcast_bytes(bytes(range(128)) if rank == 0 else None)
        tmax = max_over_ranks(float(rank + 1))
        tsum = sum_over_ranks(float(rank + 1))
        if rank == 0:
            codes = np.concatenate([bufs[r][:int(sizes[r].item())].numpy() for r in range(world)]).astype(np.int8)
            np.savez(os.path.join(out_dir, "r0.npz"), scales=s, codes=codes, sums=sums.numpy(),
                     maxes=maxes.numpy(), uid=np.frombuffer(uid, np.uint8), tmax=tmax, tsum=tsum)
        else:
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), uid=np.frombuffer(uid, np.uint8), tmax=tmax)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T,D,kind", [(513, 96, 1), (1000, 40, 0), (7, 13, 2)])
def test_token_sharding_world2_matches_unsharded(orc, tmp_path, T, D, kind):
    world, nq = 2, 5
    mp.spawn(_worker, args=(world, _free_port(), T, D, nq, kind, str(tmp_path)), nprocs=world, join=True)
    r0 = np.load(tmp_path / "r0.npz")
    r1 = np.load(tmp_path / "r1.npz")
    K = orc.fill(T, D, orc.SEED_K, kind)
    s, q, Kh = orc.roundtrip(K)
    assert np.array_equal(r0["scales"].view(np.uint32), s.view(np.uint32))  # bit-exact
    assert np.array_equal(r0["codes"].reshape(T, D), q)
    ss, mx = orc.recon_errors(K, Kh)
    attn = orc.attention_abs_sum(orc.fill(nq, D, orc.SEED_Q), K, Kh)
    sums = r0["sums"]
    assert sums[0] == pytest.approx(ss, rel=1e-12)
    assert sums[1] == pytest.approx(attn, rel=1e-12)
    assert sums[2] == T * D and sums[3] == nq * T
    assert r0["maxes"][0] == mx
    assert bytes(r0["uid"]) == bytes(r1["uid"]) == bytes(range(128))
    assert float(r0["tmax"]) == float(r1["tmax"]) == 2.0
    assert float(r0["tsum"]) == 3.0


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("T", [1, 7, 8, 131072, 131073])
def test_shard_rows_partition(world, T):
    spans = [shard_rows(T, world, r) for r in range(world)]
    assert spans[0][0] == 0
    for (a, n), (b, _) in zip(spans, spans[1:]):
        assert a + n == b
    assert sum(n for _, n in spans) == T
    assert max(n for _, n in spans) - min(n for _, n in spans) <= 1
    with pytest.raises(ValueError):
        shard_rows(T, world, world)


def _append_worker(rank, world, port, D, steps, out_dir):
    """NEXT-4 on a token-sharded cache: every rank appends its own tokens each
    step (0 allowed), the running column max is all-reduced (MAX) each step, and a
    rank re-quantizes its old rows in columns whose global scale changed -- the
    algorithm kvq_append runs with a communicator, with the oracle as the kernels."""
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(100 + rank)
        K = np.zeros((0, D), np.float32)
        absmax = np.zeros(D, np.float32)
        scales = np.zeros(D, np.float32)
        codes = np.zeros((0, D), np.int8)
        for step, n in enumerate(steps[rank]):
            new = (oracle.fill(n, D, 1000 + 10 * step + rank, 1) * (1.0 + step)).astype(np.float32)
            K = np.concatenate([K, new])
            oracle.absmax_rows(new, absmax)  # phase A on this rank's new rows
            bits = torch.from_numpy(absmax.view(np.int32).copy())
            dist.all_reduce(bits, op=dist.ReduceOp.MAX)
            absmax = bits.numpy().view(np.float32).copy()
            s_new = oracle.scales_from_absmax(absmax)  # phase B
            grown = s_new.view(np.uint32) != scales.view(np.uint32)
            scales = s_new
            if codes.shape[0] and grown.any():  # phase C: old rows of grown columns
                codes[:, grown] = oracle.quantize(K[:codes.shape[0]][:, grown], scales[grown])
            codes = np.concatenate([codes, oracle.quantize(new, scales)]) if n else codes
        np.save(os.path.join(out_dir, f"app_K{rank}.npy"), K)
        np.save(os.path.join(out_dir, f"app_q{rank}.npy"), codes)
        np.save(os.path.join(out_dir, f"app_s{rank}.npy"), scales)
    finally:
        dist.destroy_process_group()


def test_append_sharded_equals_batch(tmp_path):
    import oracle
    D = 24
    steps = [[5, 1, 0, 3, 1, 7], [2, 0, 4, 1, 1, 9]]
    mp.spawn(_append_worker, args=(2, _free_port(), D, steps, str(tmp_path)), nprocs=2, join=True)
    Ks = [np.load(tmp_path / f"app_K{r}.npy") for r in range(2)]
    s0, s1 = (np.load(tmp_path / f"app_s{r}.npy") for r in range(2))
    assert np.array_equal(s0.view(np.uint32), s1.view(np.uint32))
    batch_s = oracle.compute_scales(np.concatenate(Ks))  # the unsharded batch method over all tokens
    assert np.array_equal(s0.view(np.uint32), batch_s.view(np.uint32))
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"app_q{r}.npy"), oracle.quantize(Ks[r], batch_s))


def _consensus_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2601_04719_b200.dist import all_ranks_ok, make_peer
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mixed = all_ranks_ok(rank != 1)        # one rank fails -> every rank sees failure
        agree = all_ranks_ok(True)
        # peer setup is collective: here (no GPU) it fails on every rank, and every rank must raise
        # instead of one rank waiting on a peer that never signals
        try:
            make_peer(rank, world, 64)
            raised = False
        except Exception:  # noqa: BLE001
            raised = True
        np.savez(os.path.join(out_dir, f"c{rank}.npz"), mixed=mixed, agree=agree, raised=raised)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path of the collective setup")
def test_peer_setup_is_collective(tmp_path):
    world, port = 3, _free_port()
    mp.start_processes(_consensus_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        z = np.load(tmp_path / f"c{r}.npz")
        assert not bool(z["mixed"]) and bool(z["agree"]) and bool(z["raised"])
