"""Token-dimension sharding helpers.

Rank r of R owns the contiguous row block [row0, row0+rows) of the global
T x D key matrix.  The only exchange step of the method is the all-reduce MAX
of the D column maxima inside kvq_compute_scales (done by libkvq.so over NCCL);
everything here is host-side plumbing: the partition, the NCCL unique-id
bootstrap over torch.distributed, and max-over-ranks timing.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(T: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row partition: the first T % world ranks get one extra row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(T, world)
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


def broadcast_bytes(payload: bytes | None, src: int = 0, group=None) -> bytes:
    """Broadcast a short byte string (e.g. a 128-byte ncclUniqueId) from `src`
    to every rank of the default process group (works over gloo and nccl)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return payload
    obj = [payload]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (device-timed milliseconds) over all ranks."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def max_over_ranks_vec(xs, device=None) -> list:
    """Element-wise max over all ranks of a per-rank list of scalars (per-step device times)."""
    xs = [float(x) for x in xs]
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return xs
    t = torch.tensor(xs, dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def sum_over_ranks(x: float, device=None) -> float:
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def make_comm(rank: int, world: int):
    """Create the library's NCCL communicator: rank 0 draws the unique id, the
    default process group broadcasts it, every rank calls kvq_comm_init."""
    from .kvq import Comm, kvq_comm_unique_id
    uid = kvq_comm_unique_id() if rank == 0 else None
    uid = broadcast_bytes(uid, src=0)
    return Comm(uid, world, rank)


def all_ranks_ok(ok: bool) -> bool:
    """True iff `ok` on every rank of the default process group (MIN all-reduce)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return ok
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def enable_nvls(peer, rank: int, world: int) -> bool:
    """Route the peer's a7 exchange through NVLS multicast (multimem.ld_reduce in the NVSwitch) when every
    rank can: rank 0 creates the multicast object and broadcasts its handle, every rank joins, then (all
    joined) maps, then (all mapped) enables.  Any failure anywhere: every rank releases the multicast
    resources and keeps the P2P exchange.  Returns whether NVLS is active (the same on every rank)."""
    blob, ok = None, True
    peer.nvls_reason = ""
    if rank == 0:
        try:
            blob = peer.nvls_create()
        except Exception as e:  # noqa: BLE001  (no multicast on this device / driver)
            blob = None
            peer.nvls_reason = str(e)
    blob = broadcast_bytes(blob, src=0)
    ok = blob is not None
    if ok:
        try:
            peer.nvls_join(blob)
        except Exception as e:  # noqa: BLE001
            ok = False
            peer.nvls_reason = str(e)
    ok = all_ranks_ok(ok)
    if ok:  # binding blocks until every device has joined: only once all have
        try:
            peer.nvls_map()
        except Exception as e:  # noqa: BLE001
            ok = False
            peer.nvls_reason = str(e)
        ok = all_ranks_ok(ok)
    peer.nvls_enable(ok)
    return ok


def make_peer(rank: int, world: int, D: int):
    """Create the library's peer-memory exchange (kvq_compute_scales_peer / kvq_comm_from_peer):
    every rank allocates its buffer, the default process group all-gathers the CUDA IPC handles,
    every rank maps the others'.  Collective: if any rank fails, every rank raises (so all of
    them can fall back to NCCL together instead of waiting on a peer that never signals)."""
    from .kvq import Peer
    p, handle, err = None, b"", None
    try:
        p = Peer(world, rank, D)
        handle = p.ipc_handle
    except Exception as e:  # noqa: BLE001
        err = e
    handles = [None] * world
    dist.all_gather_object(handles, handle)
    if err is None and all(handles):
        try:
            p.open(handles)
        except Exception as e:  # noqa: BLE001
            err = e
    elif err is None:
        err = RuntimeError("kvq peer setup failed on another rank")
    if not all_ranks_ok(err is None):
        if p is not None:
            p.destroy()
        raise err if err is not None else RuntimeError("kvq peer setup failed on another rank")
    return p
