"""GPU parity of the INT4 / INT2 packed variant (NEXT-3; reading Q19) against the
oracle: scales, packed code bytes and K_hat bit-exact, on the vector path
(D % (32/bits) == 0, aligned) and the scalar path (any D), fused and separate."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FMT = {4: 2, 2: 3}


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


def gpu_rt(kvq, K, bits, fused):
    Kd = dev(K)
    s = kvq.kvq_compute_scales_fmt(Kd, FMT[bits])
    if fused:
        p, kh = kvq.kvq_quantize_packed(Kd, s, bits, want_khat=True)
    else:
        p = kvq.kvq_quantize_packed(Kd, s, bits)
        kh = kvq.kvq_dequantize_packed(p, s, K.shape[1], bits)
    return host(s), host(p), host(kh)


@pytest.mark.parametrize("bits", [4, 2])
@pytest.mark.parametrize("shape", [(1, 1), (3, 7), (64, 128), (1000, 13), (129, 1024), (33, 4096), (17, 48), (5, 200)])
@pytest.mark.parametrize("dist", [0, 1])
@pytest.mark.parametrize("fused", [False, True])
def test_lowbit_bit_exact(kvq, orc, bits, shape, dist, fused):
    K = orc.fill(*shape, 31, dist)
    s, p, kh = gpu_rt(kvq, K, bits, fused)
    so, po, kho = orc.roundtrip_q(K, bits)
    same_bits(s, so)
    same_bits(p, po)
    same_bits(kh, kho)


@pytest.mark.parametrize("bits", [4, 2])
@pytest.mark.parametrize("name", ["zeros", "negzero", "subnormal", "ties", "mixed", "underflow_col"])
def test_lowbit_structured(kvq, orc, bits, name):
    rng = np.random.default_rng(3)
    T, D = 96, 32
    if name == "zeros":
        K = np.zeros((T, D), np.float32)
    elif name == "negzero":
        K = np.full((T, D), -0.0, np.float32)
        K[3, :] = 0.5
    elif name == "subnormal":
        K = (rng.uniform(-1, 1, (T, D)) * 2.0 ** -140).astype(np.float32)
    elif name == "ties":  # quotients at half-integers (max row fixes s = 1 for INT4: max 7; INT2: max 1)
        vals = (np.array([7, 0.5, 1.5, 2.5, -0.5, -1.5, 6.5, -6.5], np.float32) if bits == 4 else
                np.array([1, 0.5, -0.5, 0.25, -0.75, 0.75, 1, -1], np.float32))
        K = np.tile(vals[:, None], (12, D)).astype(np.float32)
    elif name == "underflow_col":  # a column whose max/qmax underflows to a subnormal or zero scale
        K = rng.uniform(-1, 1, (T, D)).astype(np.float32)
        K[:, 5] = (rng.uniform(-1, 1, T) * 2.0 ** -147).astype(np.float32)
        K[:, 6] = 0.0
    else:
        K = (rng.uniform(-1, 1, (T, D)) * 2.0 ** rng.integers(-60, 60, (T, D))).astype(np.float32)
    for fused in (False, True):
        s, p, kh = gpu_rt(kvq, K, bits, fused)
        so, po, kho = orc.roundtrip_q(K, bits)
        same_bits(s, so)
        same_bits(p, po)
        same_bits(kh, kho)


@pytest.mark.parametrize("bits", [4, 2])
@pytest.mark.parametrize("scale", [1.0, 1 / 7, 0.1, 3 * 2.0 ** -10])
def test_lowbit_exhaustive_binades(kvq, orc, bits, scale):
    """Every fp32 x with |x/s| in [2^-3, 2^4) (both signs) for a fixed s, laid out
    as rows of 32/bits columns so the vector (reciprocal + repair) path runs:
    all codes, all ties, the clamp region."""
    C = 32 // bits
    s = np.float32(scale)
    lo_b = int(np.float32(s * 0.125).view(np.uint32))
    hi_b = int(np.float32(s * 16).view(np.uint32))
    for c0 in range(lo_b, hi_b, 1 << 24):
        x = np.arange(c0, min(c0 + (1 << 24), hi_b), dtype=np.uint32).view(np.float32)
        x = np.concatenate([x, -x])
        x = np.concatenate([x, np.zeros((-len(x)) % C, np.float32)]).reshape(-1, C)
        sv = np.full(C, s, np.float32)
        p, kh = kvq.kvq_quantize_packed(dev(x), dev(sv), bits, want_khat=True)
        qo = orc.quantize_q(x, sv, bits)
        same_bits(host(p), orc.pack_codes(qo, bits))
        same_bits(host(kh), orc.dequantize(qo, sv))


@pytest.mark.parametrize("bits", [4, 2])
def test_lowbit_metrics(kvq, orc, bits):
    """Low-bit reconstruction through the fidelity checks (a5, a6) vs the oracle."""
    T, D, nq = 2048, 1024, 64
    K = orc.fill(T, D)
    Q = orc.fill(nq, D, 43)
    Kd = dev(K)
    s = kvq.kvq_compute_scales_fmt(Kd, FMT[bits])
    p, kh = kvq.kvq_quantize_packed(Kd, s, bits, want_khat=True)
    m = kvq.kvq_error_metrics(Kd, kh, dev(Q), s)
    so, po, kho = orc.roundtrip_q(K, bits)
    same_bits(host(kh), kho)
    ss, mx = orc.recon_errors(K, kho)
    assert abs(m["sum_sq"] - ss) <= 1e-5 * ss and m["max_abs"] == mx
    attn = orc.attention_error(Q, K, kho)
    assert abs(m["attn_mean_abs"] - attn) <= 1e-5 * attn
    assert mx <= float(so.max()) * (0.5 + 2.0 ** -16)


def test_packed_api_errors(kvq):
    K = torch.zeros((4, 8), dtype=torch.float32, device="cuda")
    s = torch.ones(8, dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        kvq.kvq_packed_row_bytes(8, 3)
    from paper_2601_04719_b200._lib import check
    with pytest.raises(kvq.KvqError):
        check(kvq.load().kvq_quantize_packed(K.data_ptr(), s.data_ptr(), 4, 8, 3, K.data_ptr(), None, None), "x")
