"""GPU parity at the extremes of BASELINE config C5 (2^20..2^30 elements, head_dim 128/1024/8192, single-pass
fused vs two-pass kernels): kvq_quantize_fused as dispatched and with the single pass forced, and the
separate kvq_compute_scales + kvq_quantize + kvq_dequantize, against the SHA-256 of the oracle's scales,
codes and K_hat (tests/golden/oracle_c5.json, written by scripts/oracle_c5_goldens.py from oracle/ only and
pinned by numpy in tests/test_oracle_pins.py).  Bit-exact: Alg. 1, Eq. 6-8 with readings Q1-Q8."""
import hashlib
import json
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_c5.json")))
SHAPES = [k for k in GOLD if not k.startswith("_")]


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_04719_b200 import kvq as k
    k.kvq_device_check()
    return k


def sha(t, chunk_rows=1 << 14):
    """sha256 of a CUDA tensor's row-major bytes, copied to the host in row chunks."""
    torch.cuda.synchronize()
    h = hashlib.sha256()
    flat = t.reshape(t.shape[0], -1)
    for r0 in range(0, flat.shape[0], chunk_rows):
        h.update(flat[r0:r0 + chunk_rows].cpu().numpy().tobytes())
    return h.hexdigest()


@pytest.mark.timeout(900)
@pytest.mark.parametrize("path", ["fused", "fused_single", "separate"])
@pytest.mark.parametrize("name", SHAPES)
def test_c5_extremes_bit_exact(kvq, monkeypatch, name, path):
    g = GOLD[name]
    T, D = g["T"], g["D"]
    K = kvq.kvq_synth_fill(T, D, seed=42)
    if path == "separate":
        s = kvq.kvq_compute_scales(K)
        q = kvq.kvq_quantize(K, s)
        kh = kvq.kvq_dequantize(q, s)
    else:
        if path == "fused_single":
            monkeypatch.setenv("KVQ_FUSED_FORCE_SINGLE", "1")
        s, q, kh, single = kvq.kvq_quantize_fused(K)
        if path == "fused_single":
            assert single, "the single cooperative pass must take this shape"
    assert sha(s.view(1, -1)) == g["scales_sha256"]
    assert sha(q) == g["codes_sha256"]
    assert sha(kh) == g["k_hat_sha256"]
    del K, q, kh
    torch.cuda.empty_cache()
