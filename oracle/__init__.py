"""CPU oracle for per-channel INT8 KV-key quantization (arxiv 2601.04719).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product (``paper_2601_04719_b200``) never imports it and shares
no code with it; ``kvq_oracle.c`` is the arithmetic, this module only marshals
numpy arrays into it via ctypes and streams large matrices in row blocks.

Every function cites the passage it follows in kvq_oracle.c.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kvq_oracle.c")
_LIB = os.path.join(_HERE, "libkvq_oracle.so")
CFLAGS = ["-O2", "-std=c99", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared"]

SEED_K = 42
SEED_Q = 43
DIST_UNIFORM, DIST_OUTLIER, DIST_ONGRID = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile kvq_oracle.c with gcc (plain C99, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i64, u64, vp, dp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)
        L.kvqo_splitmix64.restype = u64
        L.kvqo_splitmix64.argtypes = [u64, u64]
        L.kvqo_uniform.restype = ctypes.c_float
        L.kvqo_uniform.argtypes = [u64, u64]
        L.kvqo_fill.argtypes = [vp, i64, i64, i64, u64, ctypes.c_int]
        L.kvqo_compute_scales.argtypes = [vp, i64, i64, vp]
        L.kvqo_absmax_rows.argtypes = [vp, i64, i64, vp]
        L.kvqo_scales_from_absmax.argtypes = [vp, i64, vp]
        L.kvqo_quantize.argtypes = [vp, vp, i64, i64, vp]
        L.kvqo_dequantize.argtypes = [vp, vp, i64, i64, vp]
        L.kvqo_recon_errors.argtypes = [vp, vp, i64, dp, dp]
        L.kvqo_scores.argtypes = [vp, i64, vp, i64, i64, vp]
        L.kvqo_attention_abs_sum.restype = ctypes.c_double
        L.kvqo_attention_abs_sum.argtypes = [vp, i64, vp, vp, i64, i64]
        L.kvqo_theoretical_max.restype = ctypes.c_double
        L.kvqo_theoretical_max.argtypes = [vp, i64]
        L.kvqo_e4m3_decode.restype = ctypes.c_float
        L.kvqo_e4m3_decode.argtypes = [ctypes.c_uint8]
        L.kvqo_e4m3_encode.restype = ctypes.c_uint8
        L.kvqo_e4m3_encode.argtypes = [ctypes.c_float]
        L.kvqo_scales_from_absmax_e4m3.argtypes = [vp, i64, vp]
        L.kvqo_quantize_e4m3.argtypes = [vp, vp, i64, i64, vp]
        L.kvqo_dequantize_e4m3.argtypes = [vp, vp, i64, i64, vp]
        L.kvqo_scales_from_absmax_q.argtypes = [vp, i64, ctypes.c_int, vp]
        L.kvqo_quantize_q.argtypes = [vp, vp, i64, i64, ctypes.c_int, vp]
        L.kvqo_pack_codes.argtypes = [vp, i64, i64, ctypes.c_int, vp]
        L.kvqo_unpack_codes.argtypes = [vp, i64, i64, ctypes.c_int, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# --------------------------------------------------------------------------- generator
def splitmix64(seed: int, i: int) -> int:
    return int(lib().kvqo_splitmix64(seed, i))


def uniform(seed: int, i: int) -> float:
    return float(lib().kvqo_uniform(seed, i))


def fill(T: int, D: int, seed: int = SEED_K, dist: int = DIST_UNIFORM, row0: int = 0) -> np.ndarray:
    """Rows [row0, row0+T) of the seeded synthetic matrix."""
    out = np.empty((T, D), dtype=np.float32)
    lib().kvqo_fill(_p(out), row0, T, D, seed, dist)
    return out


# --------------------------------------------------------------------------- the method
def compute_scales(K) -> np.ndarray:
    """Alg. 1 / Listing 2."""
    K = _f32(K)
    T, D = K.shape
    s = np.empty(D, dtype=np.float32)
    lib().kvqo_compute_scales(_p(K), T, D, _p(s))
    return s


def absmax_rows(K, max_abs: np.ndarray) -> None:
    K = _f32(K)
    lib().kvqo_absmax_rows(_p(K), K.shape[0], K.shape[1], _p(max_abs))


def scales_from_absmax(max_abs: np.ndarray) -> np.ndarray:
    s = np.empty_like(max_abs)
    lib().kvqo_scales_from_absmax(_p(max_abs), max_abs.shape[0], _p(s))
    return s


def quantize(K, scales) -> np.ndarray:
    """Eq. 7 / Listing 3 with readings Q1, Q2, Q4, Q5."""
    K = _f32(K)
    scales = _f32(scales)
    T, D = K.shape
    assert scales.shape == (D,)
    q = np.empty((T, D), dtype=np.int8)
    lib().kvqo_quantize(_p(K), _p(scales), T, D, _p(q))
    return q


def dequantize(q, scales) -> np.ndarray:
    """Eq. 8 / Listing 4."""
    q = np.ascontiguousarray(q, dtype=np.int8)
    scales = _f32(scales)
    T, D = q.shape
    out = np.empty((T, D), dtype=np.float32)
    lib().kvqo_dequantize(_p(q), _p(scales), T, D, _p(out))
    return out


def recon_errors(A, B, state=None):
    """(sum_sq, max_abs) accumulated in double (reading Q9)."""
    A = _f32(A).reshape(-1)
    B = _f32(B).reshape(-1)
    ss = ctypes.c_double(0.0 if state is None else state[0])
    mx = ctypes.c_double(0.0 if state is None else state[1])
    lib().kvqo_recon_errors(_p(A), _p(B), A.shape[0], ctypes.byref(ss), ctypes.byref(mx))
    return ss.value, mx.value


def l2_error(A, B) -> float:
    return float(np.sqrt(recon_errors(A, B)[0]))


def max_abs_error(A, B) -> float:
    return recon_errors(A, B)[1]


def scores(Q, K) -> np.ndarray:
    """S = Q K^T, raw dot products in double (reading Q10)."""
    Q = _f32(Q)
    K = _f32(K)
    S = np.empty((Q.shape[0], K.shape[0]), dtype=np.float64)
    lib().kvqo_scores(_p(Q), Q.shape[0], _p(K), K.shape[0], K.shape[1], _p(S))
    return S


def attention_abs_sum(Q, K, K_hat) -> float:
    Q, K, K_hat = _f32(Q), _f32(K), _f32(K_hat)
    return float(lib().kvqo_attention_abs_sum(_p(Q), Q.shape[0], _p(K), _p(K_hat), K.shape[0], K.shape[1]))


def attention_error(Q, K, K_hat) -> float:
    """mean_{i,t} |q_i.k_t - q_i.khat_t| (readings Q10, Q11)."""
    return attention_abs_sum(Q, K, K_hat) / (Q.shape[0] * K.shape[0])


def theoretical_max(scales) -> float:
    scales = _f32(scales)
    return float(lib().kvqo_theoretical_max(_p(scales), scales.shape[0]))


# --------------------------------------------------------------------------- FP8 E4M3 variant (NEXT-1)
def e4m3_decode(c: int) -> float:
    return float(lib().kvqo_e4m3_decode(c))


def e4m3_encode(v: float) -> int:
    return int(lib().kvqo_e4m3_encode(v))


def compute_scales_e4m3(K) -> np.ndarray:
    """s_d = max_t |K[t,d]| / 448 (Alg. 1's max, E4M3 range; reading Q17)."""
    K = _f32(K)
    m = np.zeros(K.shape[1], dtype=np.float32)
    absmax_rows(K, m)
    s = np.empty_like(m)
    lib().kvqo_scales_from_absmax_e4m3(_p(m), m.shape[0], _p(s))
    return s


def quantize_e4m3(K, scales) -> np.ndarray:
    K, scales = _f32(K), _f32(scales)
    T, D = K.shape
    q = np.empty((T, D), dtype=np.uint8)
    lib().kvqo_quantize_e4m3(_p(K), _p(scales), T, D, _p(q))
    return q


def dequantize_e4m3(q, scales) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.uint8)
    scales = _f32(scales)
    T, D = q.shape
    out = np.empty((T, D), dtype=np.float32)
    lib().kvqo_dequantize_e4m3(_p(q), _p(scales), T, D, _p(out))
    return out


def roundtrip_e4m3(K):
    s = compute_scales_e4m3(K)
    q = quantize_e4m3(K, s)
    return s, q, dequantize_e4m3(q, s)


# --------------------------------------------------------------------------- INT4 / INT2 variant (NEXT-3)
QMAX = {8: 127, 4: 7, 2: 1}


def packed_row_bytes(D: int, bits: int) -> int:
    per = 8 // bits
    return (D + per - 1) // per


def compute_scales_q(K, bits: int) -> np.ndarray:
    """s_d = max_t |K[t,d]| / qmax(bits) (Alg. 1's max; reading Q19)."""
    K = _f32(K)
    m = np.zeros(K.shape[1], dtype=np.float32)
    absmax_rows(K, m)
    s = np.empty_like(m)
    lib().kvqo_scales_from_absmax_q(_p(m), m.shape[0], QMAX[bits], _p(s))
    return s


def quantize_q(K, scales, bits: int) -> np.ndarray:
    """Unpacked int8 codes in [-qmax, qmax]."""
    K, scales = _f32(K), _f32(scales)
    T, D = K.shape
    q = np.empty((T, D), dtype=np.int8)
    lib().kvqo_quantize_q(_p(K), _p(scales), T, D, QMAX[bits], _p(q))
    return q


def pack_codes(q, bits: int) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.int8)
    T, D = q.shape
    out = np.empty((T, packed_row_bytes(D, bits)), dtype=np.uint8)
    lib().kvqo_pack_codes(_p(q), T, D, bits, _p(out))
    return out


def unpack_codes(p, D: int, bits: int) -> np.ndarray:
    p = np.ascontiguousarray(p, dtype=np.uint8)
    T = p.shape[0]
    q = np.empty((T, D), dtype=np.int8)
    lib().kvqo_unpack_codes(_p(p), T, D, bits, _p(q))
    return q


def roundtrip_q(K, bits: int):
    """scales, packed codes, reconstruction (Eq. 8 on the unpacked codes)."""
    s = compute_scales_q(K, bits)
    q = quantize_q(K, s, bits)
    return s, pack_codes(q, bits), dequantize(q, s)


# --------------------------------------------------------------------------- whole pipeline
def roundtrip(K):
    """scales -> codes -> reconstruction for an in-memory matrix."""
    s = compute_scales(K)
    q = quantize(K, s)
    return s, q, dequantize(q, s)


def streamed_pipeline(T: int, D: int, seed: int = SEED_K, dist: int = DIST_UNIFORM,
                      block_rows: int = 4096, nq: int = 0, attn_rows: int = 0,
                      hashes: bool = True, time_budget_s: float | None = None):
    """Run the oracle over the seeded T x D matrix in row blocks (so C4's 4.3 GB
    never has to be resident) and return scales, SHA-256 of the codes and of
    K_hat (raw little-endian row-major bytes, as SURVEY Appendix), L2, max_abs
    and — over the first ``attn_rows`` rows, with nq seeded queries — the
    attention-error sum.  Two passes over the generator: pass 1 is Alg. 1,
    pass 2 quantizes, dequantizes and measures each block."""
    max_abs = np.zeros(D, dtype=np.float32)
    for r0 in range(0, T, block_rows):
        absmax_rows(fill(min(block_rows, T - r0), D, seed, dist, r0), max_abs)
    s = scales_from_absmax(max_abs)
    hq, hk = hashlib.sha256(), hashlib.sha256()
    state = (0.0, 0.0)
    Q = fill(nq, D, SEED_Q) if nq else None
    attn_sum = 0.0
    for r0 in range(0, T, block_rows):
        K = fill(min(block_rows, T - r0), D, seed, dist, r0)
        q = quantize(K, s)
        Kh = dequantize(q, s)
        if hashes:
            hq.update(q.tobytes())
            hk.update(Kh.tobytes())
        state = recon_errors(K, Kh, state)
        if nq and r0 < attn_rows:
            n = min(K.shape[0], attn_rows - r0)
            attn_sum += attention_abs_sum(Q, K[:n], Kh[:n])
    out = dict(scales=s, l2=float(np.sqrt(state[0])), sum_sq=state[0], max_abs=state[1],
               theoretical_max=theoretical_max(s),
               scales_sha=hashlib.sha256(s.tobytes()).hexdigest(),
               q_sha=hq.hexdigest() if hashes else None, khat_sha=hk.hexdigest() if hashes else None)
    if nq:
        out["attn_abs_sum"] = attn_sum
        out["attn_mean_abs"] = attn_sum / (nq * min(T, attn_rows))
    return out


def time_pipeline(T: int, D: int, rows: int, seed: int = SEED_K):
    """Time the oracle's scales + quantize + dequantize on the first ``rows``
    rows of the T x D workload (a bounded sample; generation excluded).
    Returns (seconds, elements)."""
    K = fill(rows, D, seed)
    t0 = time.perf_counter()
    s = compute_scales(K)
    q = quantize(K, s)
    dequantize(q, s)
    return time.perf_counter() - t0, rows * D
