"""ctypes loader for libkvq.so (the C ABI in include/kvq.h and include/kvq_synth.h).

Argument marshalling only.  There is no fallback: if the shared library is
missing and cannot be built, importing the binding raises.
"""
from __future__ import annotations

import ctypes
import os

from . import build as _build

LIB_PATH = _build.LIB

# kvq_status
OK, ERR_INVALID_VALUE, ERR_CUDA, ERR_NCCL, ERR_UNSUPPORTED = 0, 1, 2, 3, 4
STATUS_NAMES = {0: "KVQ_OK", 1: "KVQ_ERR_INVALID_VALUE", 2: "KVQ_ERR_CUDA", 3: "KVQ_ERR_NCCL",
                4: "KVQ_ERR_UNSUPPORTED"}


class kvq_metrics(ctypes.Structure):
    _fields_ = [("l2", ctypes.c_double), ("max_abs", ctypes.c_double), ("attn_mean_abs", ctypes.c_double),
                ("theoretical_max", ctypes.c_double), ("sum_sq", ctypes.c_double),
                ("attn_abs_sum", ctypes.c_double), ("n_elems", ctypes.c_int64), ("n_scores", ctypes.c_int64)]

    def to_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# (name, restype, argtypes) for every exported symbol; tests check this list
# against the declarations in include/*.h.
_i64, _u64, _vp, _int, _sz = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
SIGNATURES = {
    "kvq_abi_version": (_int, []),
    "kvq_status_string": (ctypes.c_char_p, [_int]),
    "kvq_last_error": (ctypes.c_char_p, []),
    "kvq_device_check": (_int, []),
    "kvq_comm_unique_id": (_int, [_vp]),
    "kvq_comm_init": (_int, [ctypes.POINTER(_vp), _vp, _int, _int]),
    "kvq_comm_destroy": (_int, [_vp]),
    "kvq_compute_scales": (_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "kvq_compute_scales_fmt": (_int, [_vp, _i64, _i64, _vp, _int, _vp, _vp]),
    "kvq_quantize_e4m3": (_int, [_vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "kvq_dequantize_e4m3": (_int, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "kvq_append_workspace_size": (_sz, [_i64]),
    "kvq_append": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _vp]),
    "kvq_packed_row_bytes": (_i64, [_i64, _int]),
    "kvq_quantize_packed": (_int, [_vp, _vp, _i64, _i64, _int, _vp, _vp, _vp]),
    "kvq_dequantize_packed": (_int, [_vp, _vp, _i64, _i64, _int, _vp, _vp]),
    "kvq_quantize": (_int, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "kvq_dequantize": (_int, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "kvq_quantize_dequantize": (_int, [_vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "kvq_quantize_fused_workspace_size": (_sz, [_i64, _i64]),
    "kvq_quantize_fused": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _sz, _vp, ctypes.POINTER(_int), _vp]),
    "kvq_error_metrics_workspace_size": (_sz, [_i64, _i64, _i64]),
    "kvq_error_metrics_async": (_int, [_vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _sz, _vp, _vp, _vp]),
    "kvq_error_metrics": (_int, [_vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _sz, _vp,
                                 ctypes.POINTER(kvq_metrics), _vp]),
    "kvq_roundtrip_workspace_size": (_sz, [_i64, _i64, _i64]),
    "kvq_roundtrip": (_int, [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _i64, _vp, _sz, _vp, _vp, _vp]),
    "kvq_step_workspace_size": (_sz, [_i64, _i64, _i64]),
    "kvq_step": (_int, [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp, _vp, _vp]),
    "kvq_attention_scores_workspace_size": (_sz, [_i64, _i64]),
    "kvq_attention_scores": (_int, [_vp, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    "kvq_scores_from_codes_workspace_size": (_sz, [_i64, _i64]),
    "kvq_scores_from_codes": (_int, [_vp, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    "kvq_roundtrip_host_workspace_size": (_sz, [_i64, _i64, _i64]),
    "kvq_roundtrip_host": (_int, [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _vp, ctypes.POINTER(kvq_metrics), _vp,
                                  _sz, _vp, _vp]),
    "kvq_roundtrip_host_async": (_int, [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _vp]),
    "kvq_synth_fill": (_int, [_vp, _i64, _i64, _i64, _u64, _int, _vp]),
    "kvq_peer_handle_bytes": (_sz, []),
    "kvq_comm_from_peer": (_int, [ctypes.POINTER(_vp), _vp]),
    "kvq_peer_init": (_int, [ctypes.POINTER(_vp), _int, _int, _i64, _vp]),
    "kvq_peer_open": (_int, [_vp, _vp]),
    "kvq_peer_destroy": (_int, [_vp]),
    "kvq_peer_nvls_handle_bytes": (_sz, []),
    "kvq_peer_nvls_create": (_int, [_vp, _vp]),
    "kvq_peer_nvls_join": (_int, [_vp, _vp]),
    "kvq_peer_nvls_map": (_int, [_vp]),
    "kvq_peer_nvls_enable": (_int, [_vp, _int]),
    "kvq_peer_nvls_active": (_int, [_vp]),
    "kvq_compute_scales_peer": (_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
}

_lib = None


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load libkvq.so (building it with nvcc first if it does not exist)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if not build_if_missing:
            raise ImportError(f"{LIB_PATH} is missing; run `python -m paper_2601_04719_b200.build`")
        _build.build()
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class KvqError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {detail}")


def check(status: int, where: str) -> None:
    if status != OK:
        detail = load().kvq_last_error()
        raise KvqError(status, where, detail.decode() if detail else "")
