"""Thin Python binding of libkvq.so with the same names as the C ABI
(include/kvq.h).  Argument marshalling only: torch supplies device memory and
streams, every step of the path runs in libkvq.so's kernels.  Tensors must be
CUDA tensors on the current device (host tensors for the *_host call); there is
no CPU fallback and a missing/unsupported GPU raises KvqError.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from ._lib import KvqError, check, kvq_metrics, load

__all__ = [
    "KvqError", "Comm", "kvq_compute_scales", "kvq_quantize", "kvq_dequantize", "kvq_quantize_dequantize",
    "kvq_error_metrics", "kvq_error_metrics_async", "kvq_error_metrics_workspace_size", "kvq_attention_scores",
    "kvq_roundtrip_host", "kvq_roundtrip_host_workspace_size", "kvq_synth_fill", "kvq_device_check",
    "kvq_comm_unique_id", "METRICS_BYTES", "metrics_from_device", "kvq_roundtrip", "kvq_roundtrip_workspace_size",
    "kvq_quantize_fused", "kvq_roundtrip_host_async", "metrics_from_host", "kvq_compute_scales_fmt",
    "kvq_quantize_e4m3", "kvq_dequantize_e4m3", "FMT_INT8", "FMT_E4M3", "kvq_scores_from_codes",
    "FMT_INT4", "FMT_INT2", "kvq_packed_row_bytes", "kvq_quantize_packed", "kvq_dequantize_packed",
    "kvq_append", "kvq_append_workspace_size", "AppendCache",
]

load()  # fail loudly at import if libkvq.so cannot be loaded or built

METRICS_BYTES = ctypes.sizeof(kvq_metrics)
DIST_UNIFORM, DIST_OUTLIER, DIST_ONGRID = 0, 1, 2


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _mat(t: torch.Tensor, dtype, name: str, cuda: bool = True):
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if t.dim() != 2:
        raise ValueError(f"{name}: expected a [T, D] matrix, got shape {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous row-major")
    if cuda and not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor (there is no CPU path)")
    return t.shape[0], t.shape[1]


def _vec(t: torch.Tensor, n: int, name: str):
    if t.dtype != torch.float32 or t.numel() != n or not t.is_contiguous() or not t.is_cuda:
        raise ValueError(f"{name}: expected contiguous CUDA float32[{n}]")


def _out(t: torch.Tensor, shape, dtype, name: str, cuda: bool = True):
    """Caller-supplied output: exact shape and dtype, contiguous, on the right side (the library writes
    shape-many elements through the raw pointer; a smaller or host buffer would be overrun or faulted)."""
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if cuda and not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor")
    if not cuda and t.is_cuda:
        raise ValueError(f"{name}: must be a host tensor")
    return t


def _buf(t: torch.Tensor, nbytes: int, name: str, cuda: bool = True):
    """Caller-supplied byte buffer (workspace, metrics output): at least nbytes, contiguous, right side."""
    if not t.is_contiguous() or t.numel() * t.element_size() < nbytes:
        raise ValueError(f"{name}: need a contiguous buffer of >= {nbytes} bytes")
    if cuda != t.is_cuda:
        raise ValueError(f"{name}: must be a {'CUDA' if cuda else 'host'} tensor")
    return t


def _comm_handle(comm):
    return None if comm is None else comm.handle


# ----------------------------------------------------------------------------- utilities
def kvq_device_check() -> None:
    check(load().kvq_device_check(), "kvq_device_check")


def kvq_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(load().kvq_comm_unique_id(buf), "kvq_comm_unique_id")
    return buf.raw


class Comm:
    """Owns a kvq_comm_t (an NCCL communicator over one GPU per process)."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int):
        assert len(unique_id) == 128
        h = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(unique_id, 128)
        check(load().kvq_comm_init(ctypes.byref(h), idbuf, nranks, rank), "kvq_comm_init")
        self.handle, self.nranks, self.rank = h, nranks, rank

    @classmethod
    def from_peer(cls, peer: "Peer") -> "Comm":
        """A communicator whose collectives go through peer memory (kvq_comm_from_peer), no NCCL."""
        c = cls.__new__(cls)
        h = ctypes.c_void_p()
        check(load().kvq_comm_from_peer(ctypes.byref(h), peer.handle), "kvq_comm_from_peer")
        c.handle, c.nranks, c.rank, c.peer = h, peer.nranks, peer.rank, peer  # keeps the peer alive
        return c

    def destroy(self):
        if self.handle:
            check(load().kvq_comm_destroy(self.handle), "kvq_comm_destroy")
            self.handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class Peer:
    """Owns a kvq_peer_t: this rank's exchange buffer for kvq_compute_scales_peer (a1 + a7 + a2 in
    one kernel over peer memory).  Construct on every rank, all-gather ``handle`` (bytes), then
    call ``open(handles)`` with the handles in rank order."""

    def __init__(self, nranks: int, rank: int, D: int):
        lib = load()
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(lib.kvq_peer_handle_bytes())
        check(lib.kvq_peer_init(ctypes.byref(h), nranks, rank, D, buf), "kvq_peer_init")
        self.handle, self.nranks, self.rank, self.D = h, nranks, rank, D
        self.ipc_handle = buf.raw

    def open(self, handles) -> None:
        hb = load().kvq_peer_handle_bytes()
        assert len(handles) == self.nranks and all(len(x) == hb for x in handles)
        blob = ctypes.create_string_buffer(b"".join(handles), hb * self.nranks)
        check(load().kvq_peer_open(self.handle, blob), "kvq_peer_open")

    # NVLS (multicast) for the a7 exchange: staged collective setup, see include/kvq.h
    def nvls_create(self) -> bytes:
        buf = ctypes.create_string_buffer(load().kvq_peer_nvls_handle_bytes())
        check(load().kvq_peer_nvls_create(self.handle, buf), "kvq_peer_nvls_create")
        return buf.raw

    def nvls_join(self, blob: bytes) -> None:
        n = load().kvq_peer_nvls_handle_bytes()
        if len(blob) != n:
            raise ValueError(f"NVLS handle: expected {n} bytes")
        check(load().kvq_peer_nvls_join(self.handle, ctypes.create_string_buffer(blob, n)), "kvq_peer_nvls_join")

    def nvls_map(self) -> None:
        check(load().kvq_peer_nvls_map(self.handle), "kvq_peer_nvls_map")

    def nvls_enable(self, on: bool) -> None:
        check(load().kvq_peer_nvls_enable(self.handle, 1 if on else 0), "kvq_peer_nvls_enable")

    @property
    def nvls_active(self) -> bool:
        return bool(load().kvq_peer_nvls_active(self.handle))

    def destroy(self):
        if self.handle:
            check(load().kvq_peer_destroy(self.handle), "kvq_peer_destroy")
            self.handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def kvq_compute_scales_peer(K: torch.Tensor, peer: Peer, scales: Optional[torch.Tensor] = None,
                            stream=None) -> torch.Tensor:
    """Global scales of a token-sharded K through peer memory (no NCCL); K may have 0 rows."""
    if K.dim() != 2 or K.dtype != torch.float32 or not K.is_cuda or not K.is_contiguous():
        raise ValueError("K must be a contiguous float32 CUDA matrix")
    T, D = K.shape
    if scales is None:
        scales = torch.empty(D, dtype=torch.float32, device=K.device)
    _vec(scales, D, "scales")
    check(load().kvq_compute_scales_peer(_ptr(K) if T else None, T, D, _ptr(scales), peer.handle,
                                         _stream(stream)), "kvq_compute_scales_peer")
    return scales


# ----------------------------------------------------------------------------- the hot path
def kvq_compute_scales(K: torch.Tensor, scales: Optional[torch.Tensor] = None, comm: Optional[Comm] = None,
                       stream=None) -> torch.Tensor:
    T, D = _mat(K, torch.float32, "K")
    if scales is None:
        scales = torch.empty(D, dtype=torch.float32, device=K.device)
    _vec(scales, D, "scales")
    check(load().kvq_compute_scales(_ptr(K), T, D, _ptr(scales), _comm_handle(comm), _stream(stream)),
          "kvq_compute_scales")
    return scales


FMT_INT8, FMT_E4M3, FMT_INT4, FMT_INT2 = 0, 1, 2, 3


def kvq_compute_scales_fmt(K: torch.Tensor, fmt: int, scales: Optional[torch.Tensor] = None,
                           comm: Optional[Comm] = None, stream=None) -> torch.Tensor:
    T, D = _mat(K, torch.float32, "K")
    if scales is None:
        scales = torch.empty(D, dtype=torch.float32, device=K.device)
    _vec(scales, D, "scales")
    check(load().kvq_compute_scales_fmt(_ptr(K), T, D, _ptr(scales), fmt, _comm_handle(comm), _stream(stream)),
          "kvq_compute_scales_fmt")
    return scales


def kvq_quantize_e4m3(K: torch.Tensor, scales: torch.Tensor, Kq8: Optional[torch.Tensor] = None,
                      K_hat: Optional[torch.Tensor] = None, want_khat: bool = False, stream=None):
    """FP8 E4M3 codes (uint8, OCP e4m3fn bytes); also K_hat when given or want_khat."""
    T, D = _mat(K, torch.float32, "K")
    _vec(scales, D, "scales")
    if Kq8 is None:
        Kq8 = torch.empty((T, D), dtype=torch.uint8, device=K.device)
    _out(Kq8, (T, D), torch.uint8, "Kq8")
    if K_hat is None and want_khat:
        K_hat = torch.empty((T, D), dtype=torch.float32, device=K.device)
    if K_hat is not None:
        _out(K_hat, (T, D), torch.float32, "K_hat")
    check(load().kvq_quantize_e4m3(_ptr(K), _ptr(scales), T, D, _ptr(Kq8), _ptr(K_hat), _stream(stream)),
          "kvq_quantize_e4m3")
    return (Kq8, K_hat) if K_hat is not None else Kq8


def kvq_dequantize_e4m3(Kq8: torch.Tensor, scales: torch.Tensor, K_hat: Optional[torch.Tensor] = None,
                        stream=None) -> torch.Tensor:
    T, D = _mat(Kq8, torch.uint8, "Kq8")
    _vec(scales, D, "scales")
    if K_hat is None:
        K_hat = torch.empty((T, D), dtype=torch.float32, device=Kq8.device)
    _out(K_hat, (T, D), torch.float32, "K_hat")
    check(load().kvq_dequantize_e4m3(_ptr(Kq8), _ptr(scales), T, D, _ptr(K_hat), _stream(stream)),
          "kvq_dequantize_e4m3")
    return K_hat


def kvq_append_workspace_size(D: int) -> int:
    return int(load().kvq_append_workspace_size(D))


def kvq_append(K: torch.Tensor, T_old: int, n_new: int, absmax: torch.Tensor, scales: torch.Tensor,
               Kq: torch.Tensor, K_hat: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
               comm: Optional["Comm"] = None, stream=None) -> None:
    """NEXT-4: rows [T_old, T_old + n_new) of K are new tokens; update the running
    column max / scales and the codes (and K_hat) so they equal the batch method on
    K[0:T_old + n_new].  K, Kq, K_hat may have more rows (capacity) than T_old + n_new."""
    cap, D = _mat(K, torch.float32, "K")
    if T_old < 0 or n_new < 0 or T_old + n_new > cap:
        raise ValueError(f"kvq_append: rows [{T_old}, {T_old + n_new}) exceed the capacity {cap}")
    if absmax.dtype != torch.int32 or absmax.numel() != D or not absmax.is_cuda or not absmax.is_contiguous():
        raise ValueError(f"absmax: expected contiguous CUDA int32[{D}] (uint32 bit patterns)")
    _vec(scales, D, "scales")
    if _mat(Kq, torch.int8, "Kq") [1] != D or Kq.shape[0] < T_old + n_new:
        raise ValueError("Kq: expected int8 [>= T_old + n_new, D]")
    if K_hat is not None and (_mat(K_hat, torch.float32, "K_hat")[1] != D or K_hat.shape[0] < T_old + n_new):
        raise ValueError("K_hat: expected float32 [>= T_old + n_new, D]")
    if workspace is None:
        workspace = torch.empty(kvq_append_workspace_size(D), dtype=torch.uint8, device=K.device)
    _buf(workspace, kvq_append_workspace_size(D), "workspace")
    check(load().kvq_append(_ptr(K), T_old, n_new, D, _ptr(absmax), _ptr(scales), _ptr(Kq), _ptr(K_hat),
                            _ptr(workspace), workspace.numel() * workspace.element_size(), _comm_handle(comm),
                            _stream(stream)), "kvq_append")


class AppendCache:
    """Device buffers of a growing key cache (capacity rows x D): retained fp32 K,
    int8 codes, optional K_hat, and the running absmax / scales state that
    kvq_append maintains.  Plumbing only; every step runs in kvq_append."""

    def __init__(self, capacity: int, D: int, keep_khat: bool = True, device="cuda", comm=None):
        self.D, self.T, self.comm = D, 0, comm
        self.K = torch.empty((capacity, D), dtype=torch.float32, device=device)
        self.Kq = torch.empty((capacity, D), dtype=torch.int8, device=device)
        self.K_hat = torch.empty((capacity, D), dtype=torch.float32, device=device) if keep_khat else None
        self.absmax = torch.zeros(D, dtype=torch.int32, device=device)
        self.scales = torch.zeros(D, dtype=torch.float32, device=device)
        self.ws = torch.empty(kvq_append_workspace_size(D), dtype=torch.uint8, device=device)

    def append(self, rows: Optional[torch.Tensor], stream=None) -> None:
        n = 0 if rows is None else rows.shape[0]
        if n:
            if stream is not None:
                with torch.cuda.stream(stream):
                    self.K[self.T:self.T + n].copy_(rows, non_blocking=True)
            else:
                self.K[self.T:self.T + n].copy_(rows, non_blocking=True)
        kvq_append(self.K, self.T, n, self.absmax, self.scales, self.Kq, self.K_hat, self.ws, self.comm, stream)
        self.T += n


def kvq_packed_row_bytes(D: int, bits: int) -> int:
    n = int(load().kvq_packed_row_bytes(D, bits))
    if n < 0:
        raise ValueError(f"kvq_packed_row_bytes: bad D={D} or bits={bits}")
    return n


def kvq_quantize_packed(K: torch.Tensor, scales: torch.Tensor, bits: int, Kp: Optional[torch.Tensor] = None,
                        K_hat: Optional[torch.Tensor] = None, want_khat: bool = False, stream=None):
    """INT4 (bits=4) / INT2 (bits=2) codes packed per row (uint8 [T][ceil(D*bits/8)]);
    also K_hat when given or want_khat."""
    T, D = _mat(K, torch.float32, "K")
    _vec(scales, D, "scales")
    rb = kvq_packed_row_bytes(D, bits)
    if Kp is None:
        Kp = torch.empty((T, rb), dtype=torch.uint8, device=K.device)
    if Kp.dtype != torch.uint8 or tuple(Kp.shape) != (T, rb) or not Kp.is_contiguous() or not Kp.is_cuda:
        raise ValueError(f"Kp: expected contiguous CUDA uint8[{T}, {rb}]")
    if K_hat is None and want_khat:
        K_hat = torch.empty((T, D), dtype=torch.float32, device=K.device)
    if K_hat is not None:
        _out(K_hat, (T, D), torch.float32, "K_hat")
    check(load().kvq_quantize_packed(_ptr(K), _ptr(scales), T, D, bits, _ptr(Kp), _ptr(K_hat), _stream(stream)),
          "kvq_quantize_packed")
    return (Kp, K_hat) if K_hat is not None else Kp


def kvq_dequantize_packed(Kp: torch.Tensor, scales: torch.Tensor, D: int, bits: int,
                          K_hat: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    T, rb = _mat(Kp, torch.uint8, "Kp")
    if rb != kvq_packed_row_bytes(D, bits):
        raise ValueError(f"Kp: {rb} bytes per row, expected {kvq_packed_row_bytes(D, bits)} for D={D}, bits={bits}")
    _vec(scales, D, "scales")
    if K_hat is None:
        K_hat = torch.empty((T, D), dtype=torch.float32, device=Kp.device)
    _out(K_hat, (T, D), torch.float32, "K_hat")
    check(load().kvq_dequantize_packed(_ptr(Kp), _ptr(scales), T, D, bits, _ptr(K_hat), _stream(stream)),
          "kvq_dequantize_packed")
    return K_hat


def kvq_quantize(K: torch.Tensor, scales: torch.Tensor, Kq: Optional[torch.Tensor] = None,
                 stream=None) -> torch.Tensor:
    T, D = _mat(K, torch.float32, "K")
    _vec(scales, D, "scales")
    if Kq is None:
        Kq = torch.empty((T, D), dtype=torch.int8, device=K.device)
    _out(Kq, (T, D), torch.int8, "Kq")
    check(load().kvq_quantize(_ptr(K), _ptr(scales), T, D, _ptr(Kq), _stream(stream)), "kvq_quantize")
    return Kq


def kvq_dequantize(Kq: torch.Tensor, scales: torch.Tensor, K_hat: Optional[torch.Tensor] = None,
                   stream=None) -> torch.Tensor:
    T, D = _mat(Kq, torch.int8, "Kq")
    _vec(scales, D, "scales")
    if K_hat is None:
        K_hat = torch.empty((T, D), dtype=torch.float32, device=Kq.device)
    _out(K_hat, (T, D), torch.float32, "K_hat")
    check(load().kvq_dequantize(_ptr(Kq), _ptr(scales), T, D, _ptr(K_hat), _stream(stream)), "kvq_dequantize")
    return K_hat


def kvq_quantize_dequantize(K: torch.Tensor, scales: torch.Tensor, Kq: Optional[torch.Tensor] = None,
                            K_hat: Optional[torch.Tensor] = None, stream=None):
    T, D = _mat(K, torch.float32, "K")
    _vec(scales, D, "scales")
    if Kq is None:
        Kq = torch.empty((T, D), dtype=torch.int8, device=K.device)
    if K_hat is None:
        K_hat = torch.empty((T, D), dtype=torch.float32, device=K.device)
    _out(Kq, (T, D), torch.int8, "Kq")
    _out(K_hat, (T, D), torch.float32, "K_hat")
    check(load().kvq_quantize_dequantize(_ptr(K), _ptr(scales), T, D, _ptr(Kq), _ptr(K_hat), _stream(stream)),
          "kvq_quantize_dequantize")
    return Kq, K_hat


def kvq_quantize_fused(K: torch.Tensor, scales: Optional[torch.Tensor] = None, Kq: Optional[torch.Tensor] = None,
                       K_hat: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                       comm: Optional[Comm] = None, stream=None):
    """a1..a4 in one cooperative launch when possible.  Returns (scales, Kq, K_hat, single_pass)."""
    T, D = _mat(K, torch.float32, "K")
    if scales is None:
        scales = torch.empty(D, dtype=torch.float32, device=K.device)
    _vec(scales, D, "scales")
    if Kq is None:
        Kq = torch.empty((T, D), dtype=torch.int8, device=K.device)
    if K_hat is None:
        K_hat = torch.empty((T, D), dtype=torch.float32, device=K.device)
    _out(Kq, (T, D), torch.int8, "Kq")
    _out(K_hat, (T, D), torch.float32, "K_hat")
    need = int(load().kvq_quantize_fused_workspace_size(T, D))
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=K.device)
    _buf(workspace, need, "workspace")
    flag = ctypes.c_int(0)
    check(load().kvq_quantize_fused(_ptr(K), T, D, _ptr(scales), _ptr(Kq), _ptr(K_hat), _ptr(workspace),
                                    workspace.numel() * workspace.element_size(), _comm_handle(comm), ctypes.byref(flag),
                                    _stream(stream)),
          "kvq_quantize_fused")
    return scales, Kq, K_hat, bool(flag.value)


def kvq_error_metrics_workspace_size(T: int, D: int, nq: int) -> int:
    return int(load().kvq_error_metrics_workspace_size(T, D, nq))


def _metrics_args(K, K_hat, Q, scales, workspace):
    T, D = _mat(K, torch.float32, "K")
    _out(K_hat, (T, D), torch.float32, "K_hat")
    nq = 0
    if Q is not None:
        nq, Dq = _mat(Q, torch.float32, "Q")
        if Dq != D:
            raise ValueError("Q: expected D columns")
    if scales is not None:
        _vec(scales, D, "scales")
    need = kvq_error_metrics_workspace_size(T, D, nq)
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=K.device)
    _buf(workspace, need, "workspace")
    return T, D, nq, workspace


def kvq_error_metrics_async(K, K_hat, Q=None, scales=None, out_dev: Optional[torch.Tensor] = None,
                            workspace=None, comm: Optional[Comm] = None, stream=None) -> torch.Tensor:
    """Writes a kvq_metrics struct into `out_dev` (uint8[METRICS_BYTES] on the device), asynchronously."""
    T, D, nq, workspace = _metrics_args(K, K_hat, Q, scales, workspace)
    if out_dev is None:
        out_dev = torch.empty(METRICS_BYTES, dtype=torch.uint8, device=K.device)
    _buf(out_dev, METRICS_BYTES, "out_dev")
    check(load().kvq_error_metrics_async(_ptr(K), _ptr(K_hat), T, D, _ptr(Q), nq, _ptr(scales), _ptr(workspace),
                                         workspace.numel() * workspace.element_size(), _comm_handle(comm), _ptr(out_dev), _stream(stream)),
          "kvq_error_metrics_async")
    return out_dev


def metrics_from_device(out_dev: torch.Tensor) -> dict:
    raw = bytes(out_dev.cpu().numpy().tobytes())
    return kvq_metrics.from_buffer_copy(raw).to_dict()


def kvq_error_metrics(K, K_hat, Q=None, scales=None, workspace=None, comm: Optional[Comm] = None,
                      stream=None) -> dict:
    """Synchronous: returns the metrics as a dict (l2, max_abs, attn_mean_abs, ...)."""
    T, D, nq, workspace = _metrics_args(K, K_hat, Q, scales, workspace)
    out = kvq_metrics()
    check(load().kvq_error_metrics(_ptr(K), _ptr(K_hat), T, D, _ptr(Q), nq, _ptr(scales), _ptr(workspace),
                                   workspace.numel() * workspace.element_size(), _comm_handle(comm), ctypes.byref(out), _stream(stream)),
          "kvq_error_metrics")
    return out.to_dict()


def kvq_roundtrip_workspace_size(T: int, D: int, nq: int) -> int:
    return int(load().kvq_roundtrip_workspace_size(T, D, nq))


def kvq_roundtrip(K: torch.Tensor, scales: torch.Tensor, Q: Optional[torch.Tensor] = None,
                  Kq: Optional[torch.Tensor] = None, K_hat: Optional[torch.Tensor] = None,
                  out_dev: Optional[torch.Tensor] = None, workspace=None, comm: Optional[Comm] = None,
                  stream=None):
    """a3+a4+a5+a6 in one HBM pass.  Returns (Kq, K_hat, out_dev) with out_dev a
    device kvq_metrics (read it with metrics_from_device)."""
    T, D = _mat(K, torch.float32, "K")
    _vec(scales, D, "scales")
    nq = 0
    if Q is not None:
        nq, Dq = _mat(Q, torch.float32, "Q")
        if Dq != D:
            raise ValueError("Q: expected D columns")
    if Kq is None:
        Kq = torch.empty((T, D), dtype=torch.int8, device=K.device)
    if K_hat is None:
        K_hat = torch.empty((T, D), dtype=torch.float32, device=K.device)
    _out(Kq, (T, D), torch.int8, "Kq")
    _out(K_hat, (T, D), torch.float32, "K_hat")
    need = kvq_roundtrip_workspace_size(T, D, nq)
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=K.device)
    _buf(workspace, need, "workspace")
    if out_dev is None:
        out_dev = torch.empty(METRICS_BYTES, dtype=torch.uint8, device=K.device)
    _buf(out_dev, METRICS_BYTES, "out_dev")
    check(load().kvq_roundtrip(_ptr(K), _ptr(scales), T, D, _ptr(Kq), _ptr(K_hat), _ptr(Q), nq, _ptr(workspace),
                               workspace.numel() * workspace.element_size(), _comm_handle(comm), _ptr(out_dev),
                               _stream(stream)),
          "kvq_roundtrip")
    return Kq, K_hat, out_dev


def kvq_step_workspace_size(T: int, D: int, nq: int) -> int:
    return int(load().kvq_step_workspace_size(T, D, nq))


def kvq_step(K: torch.Tensor, Q: Optional[torch.Tensor] = None, scales: Optional[torch.Tensor] = None,
             Kq: Optional[torch.Tensor] = None, K_hat: Optional[torch.Tensor] = None,
             out_dev: Optional[torch.Tensor] = None, workspace=None, comm: Optional[Comm] = None, stream=None):
    """The whole hot path in one call (a1 + a7 + a2 scales, then a3-a6).  Returns (scales, Kq, K_hat,
    out_dev) with out_dev a device kvq_metrics (metrics_from_device)."""
    T, D = _mat(K, torch.float32, "K")
    nq = 0
    if Q is not None:
        nq, Dq = _mat(Q, torch.float32, "Q")
        if Dq != D:
            raise ValueError("Q: expected D columns")
    dev = K.device
    scales = _out(scales if scales is not None else torch.empty(D, dtype=torch.float32, device=dev), (D,),
                  torch.float32, "scales")
    Kq = _out(Kq if Kq is not None else torch.empty((T, D), dtype=torch.int8, device=dev), (T, D), torch.int8, "Kq")
    K_hat = _out(K_hat if K_hat is not None else torch.empty((T, D), dtype=torch.float32, device=dev), (T, D),
                 torch.float32, "K_hat")
    need = kvq_step_workspace_size(T, D, nq)
    workspace = _buf(workspace if workspace is not None else torch.empty(need, dtype=torch.uint8, device=dev), need,
                     "workspace")
    out_dev = _buf(out_dev if out_dev is not None else torch.empty(METRICS_BYTES, dtype=torch.uint8, device=dev),
                   METRICS_BYTES, "out_dev")
    check(load().kvq_step(_ptr(K), T, D, _ptr(Q), nq, _ptr(scales), _ptr(Kq), _ptr(K_hat), _ptr(workspace),
                          workspace.numel() * workspace.element_size(), _comm_handle(comm), _ptr(out_dev),
                          _stream(stream)), "kvq_step")
    return scales, Kq, K_hat, out_dev


def kvq_attention_scores(Q: torch.Tensor, K: torch.Tensor, K_hat: Optional[torch.Tensor] = None,
                         S: Optional[torch.Tensor] = None, workspace="auto", stream=None) -> torch.Tensor:
    """workspace="auto" allocates the tensor-core workspace; None selects the CUDA-core kernel."""
    nq, D = _mat(Q, torch.float32, "Q")
    T, D2 = _mat(K, torch.float32, "K")
    if D != D2:
        raise ValueError("Q and K: different D")
    if K_hat is not None:
        _out(K_hat, (T, D), torch.float32, "K_hat")
    if S is None:
        S = torch.empty((nq, T), dtype=torch.float32, device=K.device)
    _out(S, (nq, T), torch.float32, "S")
    if isinstance(workspace, str):
        workspace = torch.empty(int(load().kvq_attention_scores_workspace_size(D, nq)), dtype=torch.uint8,
                                device=K.device)
    nbytes = 0 if workspace is None else _buf(workspace, 0, "workspace").numel() * workspace.element_size()
    check(load().kvq_attention_scores(_ptr(Q), nq, _ptr(K), _ptr(K_hat), T, D, _ptr(S), _ptr(workspace), nbytes,
                                      _stream(stream)), "kvq_attention_scores")
    return S


def kvq_scores_from_codes(Q: torch.Tensor, Kq: torch.Tensor, scales: torch.Tensor,
                          S: Optional[torch.Tensor] = None, workspace="auto", stream=None) -> torch.Tensor:
    """S[i][t] = sum_d Q[i][d] * Kq[t][d] * scales[d] from the int8 codes (tensor cores when eligible)."""
    nq, D = _mat(Q, torch.float32, "Q")
    T, D2 = _mat(Kq, torch.int8, "Kq")
    if D != D2:
        raise ValueError("Q and Kq: different D")
    _vec(scales, D, "scales")
    if S is None:
        S = torch.empty((nq, T), dtype=torch.float32, device=Kq.device)
    _out(S, (nq, T), torch.float32, "S")
    if isinstance(workspace, str):
        workspace = torch.empty(int(load().kvq_scores_from_codes_workspace_size(D, nq)), dtype=torch.uint8,
                                device=Kq.device)
    nbytes = 0 if workspace is None else _buf(workspace, 0, "workspace").numel() * workspace.element_size()
    check(load().kvq_scores_from_codes(_ptr(Q), nq, _ptr(Kq), _ptr(scales), T, D, _ptr(S), _ptr(workspace), nbytes,
                                       _stream(stream)), "kvq_scores_from_codes")
    return S


def kvq_roundtrip_host_workspace_size(T: int, D: int, nq: int) -> int:
    return int(load().kvq_roundtrip_host_workspace_size(T, D, nq))


def kvq_roundtrip_host(K_host: torch.Tensor, Q_host: Optional[torch.Tensor] = None, scales_host=None,
                       Kq_host=None, K_hat_host=None, workspace: Optional[torch.Tensor] = None,
                       comm: Optional[Comm] = None, stream=None, device=None) -> dict:
    """End-to-end from host buffers (pin them for speed); synchronizes."""
    T, D = _mat(K_host, torch.float32, "K_host", cuda=False)
    nq = 0 if Q_host is None else _mat(Q_host, torch.float32, "Q_host", cuda=False)[0]
    device = device or torch.device("cuda", torch.cuda.current_device())
    if scales_host is None:
        scales_host = torch.empty(D, dtype=torch.float32, pin_memory=K_host.is_pinned())
    if Kq_host is None:
        Kq_host = torch.empty((T, D), dtype=torch.int8, pin_memory=K_host.is_pinned())
    # host outputs the library writes with device-to-host copies: exact size and dtype (an undersized host
    # buffer would be overrun silently)
    _out(scales_host, (D,), torch.float32, "scales_host", cuda=False)
    _out(Kq_host, (T, D), torch.int8, "Kq_host", cuda=False)
    if K_hat_host is not None:
        _out(K_hat_host, (T, D), torch.float32, "K_hat_host", cuda=False)
    need = kvq_roundtrip_host_workspace_size(T, D, nq)
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=device)
    _buf(workspace, need, "workspace")
    m = kvq_metrics()
    check(load().kvq_roundtrip_host(_ptr(K_host), T, D, _ptr(Q_host), nq, _ptr(scales_host), _ptr(Kq_host),
                                    _ptr(K_hat_host), ctypes.byref(m), _ptr(workspace),
                                    workspace.numel() * workspace.element_size(),
                                    _comm_handle(comm), _stream(stream)), "kvq_roundtrip_host")
    return {"scales": scales_host, "Kq": Kq_host, "K_hat": K_hat_host, "metrics": m.to_dict()}


def kvq_roundtrip_host_async(K_host: torch.Tensor, Q_host: Optional[torch.Tensor], scales_host: torch.Tensor,
                             Kq_host: torch.Tensor, metrics_host: torch.Tensor, workspace: torch.Tensor,
                             K_hat_host: Optional[torch.Tensor] = None, comm: Optional[Comm] = None, stream=None):
    """Asynchronous host-buffer pipeline; every host tensor must be pinned.  metrics_host is a
    pinned uint8[METRICS_BYTES] tensor (decode with metrics_from_host after synchronizing)."""
    T, D = _mat(K_host, torch.float32, "K_host", cuda=False)
    nq = 0 if Q_host is None else _mat(Q_host, torch.float32, "Q_host", cuda=False)[0]
    for t in (K_host, scales_host, Kq_host, metrics_host) + ((Q_host,) if Q_host is not None else ()):
        if not t.is_pinned():
            raise ValueError("kvq_roundtrip_host_async needs pinned host tensors")
    _out(scales_host, (D,), torch.float32, "scales_host", cuda=False)
    _out(Kq_host, (T, D), torch.int8, "Kq_host", cuda=False)
    if K_hat_host is not None:
        _out(K_hat_host, (T, D), torch.float32, "K_hat_host", cuda=False)
        if not K_hat_host.is_pinned():
            raise ValueError("kvq_roundtrip_host_async needs pinned host tensors")
    _buf(metrics_host, METRICS_BYTES, "metrics_host", cuda=False)
    _buf(workspace, kvq_roundtrip_host_workspace_size(T, D, nq), "workspace")
    check(load().kvq_roundtrip_host_async(_ptr(K_host), T, D, _ptr(Q_host), nq, _ptr(scales_host), _ptr(Kq_host),
                                          _ptr(K_hat_host), _ptr(metrics_host), _ptr(workspace),
                                          workspace.numel() * workspace.element_size(),
                                          _comm_handle(comm), _stream(stream)), "kvq_roundtrip_host_async")


def metrics_from_host(buf: torch.Tensor) -> dict:
    return kvq_metrics.from_buffer_copy(bytes(buf.numpy().tobytes()[:METRICS_BYTES])).to_dict()


def kvq_synth_fill(rows: int, D: int, row0: int = 0, seed: int = 42, dist: int = DIST_UNIFORM,
                   out: Optional[torch.Tensor] = None, device=None, stream=None) -> torch.Tensor:
    """Rows [row0, row0+rows) of the seeded synthetic matrix (include/kvq_synth.h), generated on the GPU."""
    if out is None:
        out = torch.empty((rows, D), dtype=torch.float32,
                          device=device or torch.device("cuda", torch.cuda.current_device()))
    _out(out, (rows, D), torch.float32, "out")
    check(load().kvq_synth_fill(_ptr(out), row0, rows, D, seed, dist, _stream(stream)), "kvq_synth_fill")
    return out
