"""GPU: kvq_compute_scales_peer (a1 + a7 + a2 in one kernel over peer memory, SURVEY §8(f)
NEXT-4) against the oracle.  One GPU is available, so the multi-rank test runs 2 and 3
processes on cuda:0: the CUDA IPC mapping, the P2P slot stores, the epoch flags and the
double-buffered slots are the same code as across NVLink peers (time-sliced instead of
concurrent kernels)."""
import os
import socket
import traceback

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_04719_b200 import kvq as k
    k.kvq_device_check()
    return k


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


# (T, D, seed, dist) per epoch; T is split unevenly, and one epoch gives rank 0 no rows
EPOCHS = [(1000, 256, 42, 0), (513, 1024, 7, 1), (1, 64, 9, 1), (4096, 8192, 42, 0), (300, 4, 11, 1),
          (2048, 128, 5, 0)]


def test_peer_world1_matches_compute_scales(kvq, orc):
    for T, D, seed, dist in EPOCHS:
        p = kvq.Peer(1, 0, D)
        p.open([p.ipc_handle])
        K = kvq.kvq_synth_fill(T, D, seed=seed, dist=dist)
        for _ in range(3):  # epochs 1..3 (both slot parities)
            s = kvq.kvq_compute_scales_peer(K, p)
            assert np.array_equal(host(s).view(np.uint32), orc.compute_scales(orc.fill(T, D, seed, dist)).view(np.uint32))
        p.destroy()


def test_peer_rejects_bad_args(kvq):
    p = kvq.Peer(1, 0, 64)
    with pytest.raises(RuntimeError):
        kvq.kvq_compute_scales_peer(torch.zeros(4, 64, device="cuda"), p)  # not opened yet
    p.open([p.ipc_handle])
    with pytest.raises(RuntimeError):
        kvq.kvq_compute_scales_peer(torch.zeros(4, 32, device="cuda"), p)  # D differs from init
    p.destroy()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    ok_path = os.path.join(out_dir, f"rank{rank}.txt")
    try:
        import torch.distributed as dist
        import oracle as orc
        from paper_2601_04719_b200 import kvq
        from paper_2601_04719_b200.dist import make_peer, shard_rows
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        msgs = []
        for e, (T, D, seed, dst) in enumerate(EPOCHS):
            p = make_peer(rank, world, D)
            # uneven shards; in the third epoch rank 0 has no rows at all
            if T == 1:
                row0, rows = (0, 0) if rank == 0 else (0, 1) if rank == 1 else (1, 0)
            else:
                row0, rows = shard_rows(T, world, rank)
            K = kvq.kvq_synth_fill(rows, D, row0=row0, seed=seed, dist=dst) if rows else \
                torch.empty(0, D, dtype=torch.float32, device="cuda")
            want = orc.compute_scales(orc.fill(T, D, seed, dst)).view(np.uint32)
            for it in range(3):
                s = kvq.kvq_compute_scales_peer(K, p)
                got = host(s).view(np.uint32)
                if not np.array_equal(got, want):
                    msgs.append(f"epoch {e} iter {it}: {int((got != want).sum())} scales differ")
            dist.barrier()
            p.destroy()
            dist.barrier()
        # a peer-backed communicator: every collective of scales (INT8 fused, E4M3 fused, unaligned D generic),
        # roundtrip and metrics goes through peer memory, no NCCL
        for T, D, nq in [(700, 256, 64), (333, 64, 17)]:
            p = make_peer(rank, world, D)
            comm = kvq.Comm.from_peer(p)
            row0, rows = shard_rows(T, world, rank)
            Kfull = orc.fill(T, D, 42, 1)
            K = kvq.kvq_synth_fill(rows, D, row0=row0, seed=42, dist=1)
            Q = orc.fill(nq, D, 43)
            so, qo, kho = orc.roundtrip(Kfull)
            for it in range(2):
                s = kvq.kvq_compute_scales(K, comm=comm)
                if not np.array_equal(host(s).view(np.uint32), so.view(np.uint32)):
                    msgs.append(f"comm scales T={T} D={D}")
                Kq, Kh, out = kvq.kvq_roundtrip(K, s, torch.from_numpy(Q).cuda(), comm=comm)
                m = kvq.metrics_from_device(out)
                if not (np.array_equal(host(Kq), qo[row0:row0 + rows]) and
                        np.array_equal(host(Kh).view(np.uint32), kho[row0:row0 + rows].view(np.uint32))):
                    msgs.append(f"comm roundtrip codes T={T} D={D}")
                ss, mx = orc.recon_errors(Kfull, kho)
                attn = orc.attention_error(Q, Kfull, kho)
                if m["max_abs"] != mx or abs(m["sum_sq"] - ss) > 1e-5 * ss or abs(m["attn_mean_abs"] - attn) > 1e-5 * attn:
                    msgs.append(f"comm metrics T={T} D={D}: {m} vs {ss} {mx} {attn}")
                me = kvq.kvq_error_metrics(K, Kh, torch.from_numpy(Q).cuda(), s, comm=comm)
                if me["max_abs"] != mx or abs(me["attn_mean_abs"] - attn) > 1e-5 * attn:
                    msgs.append(f"comm error_metrics T={T} D={D}")
                s8 = kvq.kvq_compute_scales_fmt(K, kvq.FMT_E4M3, comm=comm)
                if not np.array_equal(host(s8).view(np.uint32), orc.compute_scales_e4m3(Kfull).view(np.uint32)):
                    msgs.append(f"comm e4m3 scales T={T} D={D}")
            Ku = kvq.kvq_synth_fill(rows, 13, row0=row0, seed=5)  # D % 4 != 0: colmax + peer MAX kernel + finalize
            pu = make_peer(rank, world, 13)
            cu = kvq.Comm.from_peer(pu)
            su = kvq.kvq_compute_scales(Ku, comm=cu)
            if not np.array_equal(host(su).view(np.uint32), orc.compute_scales(orc.fill(T, 13, 5)).view(np.uint32)):
                msgs.append(f"comm unaligned scales T={T}")
            torch.cuda.synchronize()
            dist.barrier()
            comm.destroy()
            cu.destroy()
            p.destroy()
            pu.destroy()
            dist.barrier()
        # token-sharded streaming cache (kvq_append) over the peer communicator: after every append the global
        # scales and each rank's codes equal the batch method on the union of all ranks' rows so far
        D = 64
        p = make_peer(rank, world, D)
        comm = kvq.Comm.from_peer(p)
        Kall = orc.fill(300 * world, D, 17, 1)
        cache = kvq.AppendCache(300, D, keep_khat=True, comm=comm)
        steps = [(5, 0, 2), (1, 3, 0), (100, 7, 40), (0, 0, 0), (50, 90, 1), (1, 1, 1)]
        done = [0] * world
        for st_ in steps:
            n = st_[rank % 3]
            rows = torch.from_numpy(Kall[300 * rank + done[rank]:300 * rank + done[rank] + n]).cuda() if n else None
            cache.append(rows)
            done = [done[r] + st_[r % 3] for r in range(world)]
            union = np.concatenate([Kall[300 * r:300 * r + done[r]] for r in range(world)])
            su = orc.compute_scales(union) if union.shape[0] else np.zeros(D, np.float32)
            if not np.array_equal(host(cache.scales).view(np.uint32), su.view(np.uint32)):
                msgs.append(f"append scales after {done}")
            mine = Kall[300 * rank:300 * rank + done[rank]]
            if done[rank] and not np.array_equal(host(cache.Kq[:done[rank]]), orc.quantize(mine, su)):
                msgs.append(f"append codes after {done}")
        torch.cuda.synchronize()
        dist.barrier()
        comm.destroy()
        p.destroy()
        dist.barrier()
        dist.destroy_process_group()
        with open(ok_path, "w") as f:
            f.write("OK\n" if not msgs else "\n".join(msgs))
    except Exception:
        with open(ok_path, "w") as f:
            f.write(traceback.format_exc())


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 3])
def test_peer_multiprocess_one_gpu(kvq, tmp_path, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, str(tmp_path))) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=480)
    alive = [pr for pr in procs if pr.is_alive()]
    for pr in alive:
        pr.kill()
    assert not alive, "peer exchange did not finish (hang)"
    for r in range(world):
        txt = (tmp_path / f"rank{r}.txt").read_text()
        if "cudaIpcOpenMemHandle" in txt and "not supported" in txt:
            pytest.skip("CUDA IPC unavailable in this environment: " + txt.splitlines()[-1])
        assert txt.strip() == "OK", f"rank {r}: {txt}"
