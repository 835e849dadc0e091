"""CPU-only checks of the C-ABI library: it builds, loads, exports every symbol
that include/*.h declares, and its synchronous argument validation works
without a GPU (no compute calls)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in ("kvq.h", "kvq_synth.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(kvq_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_2601_04719_b200 import _lib
    return _lib.load()


def test_header_declares_expected_api():
    names = declared_functions()
    for n in ("kvq_compute_scales", "kvq_quantize", "kvq_dequantize", "kvq_error_metrics",
              "kvq_quantize_dequantize", "kvq_comm_init", "kvq_synth_fill", "kvq_roundtrip_host"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2601_04719_b200 import _lib
    names = declared_functions()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the binding declares a signature for every exported entry point
    assert names == set(_lib.SIGNATURES), names ^ set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    from paper_2601_04719_b200 import build
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_status_strings(lib):
    assert lib.kvq_abi_version() == 1
    assert lib.kvq_status_string(0) == b"KVQ_OK"
    assert lib.kvq_status_string(3) == b"KVQ_ERR_NCCL"


def test_argument_validation_without_gpu(lib):
    from paper_2601_04719_b200._lib import ERR_INVALID_VALUE, OK
    A = 1 << 20  # fake device addresses: never dereferenced by validation
    assert lib.kvq_compute_scales(None, 4, 4, A, None, None) == ERR_INVALID_VALUE
    assert b"NULL" in lib.kvq_last_error()
    assert lib.kvq_compute_scales(A, 0, 4, 2 * A, None, None) == ERR_INVALID_VALUE
    assert lib.kvq_compute_scales(A, 4, -1, 2 * A, None, None) == ERR_INVALID_VALUE
    assert lib.kvq_compute_scales(A, 1 << 40, 1 << 30, 2 * A, None, None) == ERR_INVALID_VALUE  # T*D > 2^62
    # aliasing: scales inside K
    assert lib.kvq_compute_scales(A, 16, 16, A + 64, None, None) == ERR_INVALID_VALUE
    assert b"alias" in lib.kvq_last_error()
    assert lib.kvq_quantize(A, 2 * A, 16, 16, A + 8, None) == ERR_INVALID_VALUE  # Kq aliases K
    assert lib.kvq_dequantize(A, 2 * A, 16, 16, A, None) == ERR_INVALID_VALUE  # K_hat aliases Kq
    assert lib.kvq_quantize_dequantize(A, 2 * A, 4, 4, 3 * A, None, None) == ERR_INVALID_VALUE
    assert lib.kvq_error_metrics_async(A, 2 * A, 4, 4, None, 3, None, 3 * A, 1 << 20, None, 4 * A,
                                       None) == ERR_INVALID_VALUE  # nq > 0 without Q
    assert lib.kvq_error_metrics_async(A, 2 * A, 4, 4, None, 0, None, 3 * A, 8, None, 4 * A,
                                       None) == ERR_INVALID_VALUE  # workspace too small
    assert lib.kvq_synth_fill(None, 0, 4, 4, 42, 0, None) == ERR_INVALID_VALUE
    assert lib.kvq_synth_fill(A, 0, 4, 4, 42, 7, None) == ERR_INVALID_VALUE
    assert lib.kvq_comm_init(None, None, 1, 0) == ERR_INVALID_VALUE
    assert lib.kvq_error_metrics_workspace_size(0, 4, 0) == 0
    assert lib.kvq_error_metrics_workspace_size(1024, 128, 64) > 0
    assert lib.kvq_roundtrip_host_workspace_size(1024, 128, 64) >= 1024 * 128 * 9
    assert OK == 0


def test_valid_arguments_fail_loudly_without_gpu(lib):
    """No CPU fallback: a compute call with no usable GPU returns an error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2601_04719_b200._lib import OK
    A = 1 << 20
    st = lib.kvq_quantize(A, 2 * A, 4, 4, 3 * A, None)
    assert st != OK
    assert lib.kvq_device_check() != OK


def test_binding_import_and_errors():
    import torch
    from paper_2601_04719_b200 import kvq
    with pytest.raises(ValueError):
        kvq.kvq_compute_scales(torch.zeros(4, 4))  # CPU tensor: no CPU path
    with pytest.raises(TypeError):
        kvq.kvq_quantize(torch.zeros(4, 4, dtype=torch.float64), torch.zeros(4))


def test_next_rows_validation_without_gpu(lib):
    """FP8 / INT4-INT2 / scores-from-codes / append entry points validate their
    arguments synchronously and fail loudly (no CPU path) when they are valid."""
    import torch
    from paper_2601_04719_b200._lib import ERR_INVALID_VALUE, OK
    A = 1 << 20
    assert lib.kvq_compute_scales_fmt(A, 4, 4, 2 * A, 9, None, None) == ERR_INVALID_VALUE  # unknown format
    assert lib.kvq_packed_row_bytes(9, 4) == 5 and lib.kvq_packed_row_bytes(9, 2) == 3
    assert lib.kvq_packed_row_bytes(9, 3) == -1 and lib.kvq_packed_row_bytes(0, 4) == -1
    assert lib.kvq_quantize_packed(A, 2 * A, 4, 8, 3, 3 * A, None, None) == ERR_INVALID_VALUE  # bits
    assert lib.kvq_quantize_packed(A, 2 * A, 4, 8, 4, A + 4, None, None) == ERR_INVALID_VALUE  # Kp aliases K
    assert lib.kvq_dequantize_packed(A, 2 * A, 4, 8, 2, A, None) == ERR_INVALID_VALUE  # K_hat aliases Kp
    assert lib.kvq_quantize_e4m3(A, 2 * A, 4, 4, A + 2, None, None) == ERR_INVALID_VALUE
    assert lib.kvq_append_workspace_size(8) >= 8 * 4 and lib.kvq_append_workspace_size(0) == 0
    ws = lib.kvq_append_workspace_size(8)
    assert lib.kvq_append(A, -1, 1, 8, 2 * A, 3 * A, 4 * A, None, 5 * A, ws, None, None) == ERR_INVALID_VALUE
    assert lib.kvq_append(A, 0, 1, 8, 2 * A, 3 * A, 4 * A, None, 5 * A, 1, None, None) == ERR_INVALID_VALUE  # ws
    assert lib.kvq_append(A, 0, 4, 8, A + 8, 3 * A, 4 * A, None, 5 * A, ws, None, None) == ERR_INVALID_VALUE  # alias
    assert lib.kvq_scores_from_codes_workspace_size(1024, 64) > 0
    if not torch.cuda.is_available():
        assert lib.kvq_quantize_packed(A, 2 * A, 4, 8, 4, 3 * A, None, None) != OK
        assert lib.kvq_append(A, 0, 1, 8, 2 * A, 3 * A, 4 * A, None, 5 * A, ws, None, None) != OK
        assert lib.kvq_scores_from_codes(A, 4, 2 * A, 3 * A, 8, 16, 4 * A, None, 0, None) != OK


def test_peer_api_validation_without_gpu(lib):
    """Peer-memory exchange (kvq_peer_*, kvq_comm_from_peer, kvq_compute_scales_peer): synchronous argument
    checks, and no silent success without a GPU."""
    import ctypes
    import torch
    from paper_2601_04719_b200._lib import ERR_INVALID_VALUE, OK
    assert lib.kvq_peer_handle_bytes() == 64  # cudaIpcMemHandle_t
    h = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(64)
    assert lib.kvq_peer_init(None, 2, 0, 64, buf) == ERR_INVALID_VALUE
    assert lib.kvq_peer_init(ctypes.byref(h), 0, 0, 64, buf) == ERR_INVALID_VALUE   # nranks
    assert lib.kvq_peer_init(ctypes.byref(h), 17, 0, 64, buf) == ERR_INVALID_VALUE  # nranks > 16
    assert lib.kvq_peer_init(ctypes.byref(h), 2, 2, 64, buf) == ERR_INVALID_VALUE   # rank
    assert lib.kvq_peer_init(ctypes.byref(h), 2, 0, 0, buf) == ERR_INVALID_VALUE    # D
    assert lib.kvq_peer_init(ctypes.byref(h), 2, 0, 64, None) == ERR_INVALID_VALUE  # handle out
    assert lib.kvq_peer_open(None, buf) == ERR_INVALID_VALUE
    assert lib.kvq_comm_from_peer(ctypes.byref(h), None) == ERR_INVALID_VALUE
    assert lib.kvq_compute_scales_peer(1 << 20, 4, 64, 2 << 20, None, None) == ERR_INVALID_VALUE
    assert lib.kvq_peer_destroy(None) == OK
    if not torch.cuda.is_available():
        assert lib.kvq_peer_init(ctypes.byref(h), 2, 0, 64, buf) != OK
