"""GPU parity of the FP8 E4M3 variant (NEXT-1; reading Q17) against the oracle:
scales, codes and K_hat bit-exact, metrics within 1e-5."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REL = 1e-5


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_04719_b200 import kvq as k
    k.kvq_device_check()
    return k


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def same_bits(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    assert a.shape == b.shape and a.dtype == b.dtype, (a.shape, b.shape, a.dtype, b.dtype)
    va = a.view(np.uint8 if a.dtype.itemsize == 1 else np.uint32)
    vb = b.view(np.uint8 if b.dtype.itemsize == 1 else np.uint32)
    bad = np.nonzero(va != vb)
    if bad[0].size:
        i = tuple(x[0] for x in bad)
        raise AssertionError(f"{bad[0].size} mismatches; first at {i}: gpu={a[i]!r} oracle={b[i]!r}")


def gpu_rt(kvq, K, fused):
    Kd = dev(K)
    s = kvq.kvq_compute_scales_fmt(Kd, kvq.FMT_E4M3)
    if fused:
        q, kh = kvq.kvq_quantize_e4m3(Kd, s, want_khat=True)
    else:
        q = kvq.kvq_quantize_e4m3(Kd, s)
        kh = kvq.kvq_dequantize_e4m3(q, s)
    return host(s), host(q), host(kh)


@pytest.mark.parametrize("shape", [(1, 1), (3, 7), (64, 128), (1000, 13), (129, 1024), (33, 4096)])
@pytest.mark.parametrize("dist", [0, 1])
@pytest.mark.parametrize("fused", [False, True])
def test_e4m3_bit_exact(kvq, orc, shape, dist, fused):
    K = orc.fill(*shape, 21, dist)
    s, q, kh = gpu_rt(kvq, K, fused)
    so, qo, kho = orc.roundtrip_e4m3(K)
    same_bits(s, so)
    same_bits(q, qo)
    same_bits(kh, kho)


@pytest.mark.parametrize("name", ["zeros", "negzero", "subnormal", "ties", "mixed"])
def test_e4m3_structured(kvq, orc, name):
    rng = np.random.default_rng(2)
    T, D = 96, 20
    if name == "zeros":
        K = np.zeros((T, D), np.float32)
    elif name == "negzero":
        K = np.full((T, D), -0.0, np.float32)
        K[3, :] = 0.5
    elif name == "subnormal":
        K = (rng.uniform(-1, 1, (T, D)) * 2.0 ** -140).astype(np.float32)
    elif name == "ties":  # quotients exactly halfway between E4M3 neighbours (s = 1 after max 448)
        vals = np.array([448, 1.0625, 1.1875, 3 * 2.0 ** -10, 2.0 ** -10, 17.0, 19.0, -1.0625], np.float32)
        K = np.tile(vals[:, None], (12, D)).astype(np.float32)
    else:
        K = (rng.uniform(-1, 1, (T, D)) * 2.0 ** rng.integers(-60, 60, (T, D))).astype(np.float32)
    for fused in (False, True):
        s, q, kh = gpu_rt(kvq, K, fused)
        so, qo, kho = orc.roundtrip_e4m3(K)
        same_bits(s, so)
        same_bits(q, qo)
        same_bits(kh, kho)


@pytest.mark.parametrize("scale", [1.0, 1 / 448, 3 * 2.0 ** -10, 2.0 ** -120])
def test_e4m3_quantize_exhaustive_binades(kvq, orc, scale):
    """Every fp32 x with |x/s| in [2^-11, 2^10) (both signs): all codes, ties,
    subnormal codes and the saturation region."""
    s = np.float32(scale)
    lo_b = int(np.float32(s * 2.0 ** -11).view(np.uint32))
    hi_b = int(np.float32(s * 2.0 ** 10).view(np.uint32))
    sd = dev(np.array([s], np.float32))
    for c0 in range(lo_b, hi_b, 1 << 25):
        x = np.arange(c0, min(c0 + (1 << 25), hi_b), dtype=np.uint32).view(np.float32)
        x = np.concatenate([x, -x]).reshape(-1, 1)
        q, kh = kvq.kvq_quantize_e4m3(dev(x), sd, want_khat=True)
        qo = orc.quantize_e4m3(x, np.array([s], np.float32))
        same_bits(host(q), qo)
        same_bits(host(kh), orc.dequantize_e4m3(qo, np.array([s], np.float32)))


def test_e4m3_metrics_and_fidelity(kvq, orc):
    """FP8 reconstruction through the fidelity checks (a5, a6) vs the oracle, and
    the expected E4M3 error level (3 mantissa bits: max error <= 2^-4 |x|)."""
    T, D, nq = 2048, 1024, 64
    K = orc.fill(T, D)
    Q = orc.fill(nq, D, 43)
    Kd = dev(K)
    s = kvq.kvq_compute_scales_fmt(Kd, kvq.FMT_E4M3)
    q, kh = kvq.kvq_quantize_e4m3(Kd, s, want_khat=True)
    m = kvq.kvq_error_metrics(Kd, kh, dev(Q), s)
    so, qo, kho = orc.roundtrip_e4m3(K)
    same_bits(host(kh), kho)
    ss, mx = orc.recon_errors(K, kho)
    assert abs(m["sum_sq"] - ss) <= REL * ss and m["max_abs"] == mx
    attn = orc.attention_error(Q, K, kho)
    assert abs(m["attn_mean_abs"] - attn) <= REL * attn
    # |x| <= 1, s ~ 1/448: the top E4M3 binade [256, 448) has spacing 32, so |x - x_hat| <= 16 s
    assert mx <= 16.0 * float(so.max()) * (1 + 1e-6)
    assert mx > 4 / 254  # FP8 (3 mantissa bits) is coarser than INT8's 1/254 at the top of the range
    assert m["attn_mean_abs"] > 0 and math.isfinite(m["attn_mean_abs"])
